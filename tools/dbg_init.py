import sys; sys.path.insert(0,'.')
import numpy as np
from paper_2605_24514_b200 import BatchedSvdEngine
rng = np.random.default_rng(41)
B, m, n, k = 1024, 48, 64, 8
a0 = rng.standard_normal((B, m, k)) @ rng.standard_normal((B, k, n)) + 0.01 * rng.standard_normal((B, m, n))
engs = [BatchedSvdEngine(a0, k, m_cap=m + 16) for _ in range(4)]
diff = []
for b in range(B):
    fs = [e.factors(b) for e in engs]
    d = max(float(np.max(np.abs(f.vt - fs[0].vt))) + float(np.max(np.abs(f.s - fs[0].s))) for f in fs)
    if d > 0: diff.append((b, d))
print("init streams differing:", len(diff), diff[:8])

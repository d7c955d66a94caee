import sys; sys.path.insert(0,'.')
import numpy as np, torch
from paper_2605_24514_b200 import BatchedSvdEngine, _lib
lib = _lib.load()
rng = np.random.default_rng(41)
B, m, n, k = 1024, 48, 64, 8
a0 = rng.standard_normal((B, m, k)) @ rng.standard_normal((B, k, n)) + 0.01 * rng.standard_normal((B, m, n))
G = int(sys.argv[1]) if len(sys.argv) > 1 else 4
mode = sys.argv[2] if len(sys.argv) > 2 else "host"
engs = [BatchedSvdEngine(a0, k, m_cap=m + 16) for _ in range(4)]
for e in engs:
    if hasattr(lib, "isvd_engine_set_groups"): _lib.check(lib.isvd_engine_set_groups(e._h.h, G))
xs = rng.standard_normal((B, n))
if mode == "dev":
    xd = torch.tensor(xs, device="cuda"); torch.cuda.synchronize()
for e in engs:
    e.row_append(xs if mode == "host" else xd)
rh = [e.scalars()[1] for e in engs]
bad = sorted(set(np.concatenate([np.nonzero(r != rh[0])[0] for r in rh])))
print(mode, "G", G, "rho diffs at", bad)
for b in bad[:3]:
    fs = [e.factors(b) for e in engs]
    print(" stream", b, "rho", [float(r[b]) for r in rh], "dvt", [float(np.max(np.abs(f.vt - fs[0].vt))) for f in fs], "ds", [float(np.max(np.abs(f.s - fs[0].s))) for f in fs])

"""Host-side cost of one e2e step (row append from pinned host rows + scalars)."""
import sys, time
from pathlib import Path
import numpy as np
import torch
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa
from paper_2605_24514_b200 import BatchedSvdEngine  # noqa

m = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 18
dev = torch.device("cuda", 0)
a0, rows = bench.make_inputs_5b(torch, dev, m=m)
eng = BatchedSvdEngine(a0, 128, m_cap=m + 300, k_cap=128)
h = torch.empty(rows.shape, dtype=torch.float64, pin_memory=True); h.copy_(rows); hr = h.numpy()
eng.synchronize()
ta = tb = tc = 0.0
for t in range(64):
    t0 = time.perf_counter()
    eng.row_append(hr[t:t + 1])
    t1 = time.perf_counter()
    eng.synchronize()
    t2 = time.perf_counter()
    eng.scalars()
    t3 = time.perf_counter()
    if t >= 8:
        ta += t1 - t0; tb += t2 - t1; tc += t3 - t2
n = 56
print(f"host issue {ta / n * 1e6:.1f} us, wait gpu {tb / n * 1e6:.1f} us, scalars {tc / n * 1e6:.1f} us")
# device-resident rows
t0 = time.perf_counter()
for t in range(64, 128):
    eng.row_append(rows[t:t + 1])
t1 = time.perf_counter()
eng.synchronize()
t2 = time.perf_counter()
print(f"device rows: host issue {(t1 - t0) / 64 * 1e6:.1f} us/step, total {(t2 - t0) / 64 * 1e6:.1f} us/step")

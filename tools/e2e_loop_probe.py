"""Per-call host timing of the 5a e2e loop (lag-1 readback)."""
import sys, time
from pathlib import Path
import numpy as np
import torch
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa
from paper_2605_24514_b200 import BatchedSvdEngine  # noqa
dev = torch.device("cuda", 0)
T = 24
a0, rows, ii, jj, dd = bench.make_inputs(torch, dev, list(range(4096)), n_events=T)
eng = BatchedSvdEngine(a0, 32, m_cap=1024 + T, k_cap=32)
hr = torch.empty(rows.shape, dtype=torch.float64, pin_memory=True); hr.copy_(rows); hr = hr.numpy()
hi = torch.empty(ii.shape, dtype=torch.int64, pin_memory=True); hi.copy_(ii); hi = hi.numpy()
hj = torch.empty(jj.shape, dtype=torch.int64, pin_memory=True); hj.copy_(jj); hj = hj.numpy()
hd = torch.empty(dd.shape, dtype=torch.float64, pin_memory=True); hd.copy_(dd); hd = hd.numpy()
res = torch.empty((2, 3 * 4096), dtype=torch.float64, pin_memory=True)
eng.synchronize()
t00 = time.perf_counter()
for t in range(T):
    t0 = time.perf_counter()
    if t % 2 == 0:
        eng.row_append(hr[t // 2])
    else:
        eng.rank_one_update(hi[t // 2], hj[t // 2], hd[t // 2])
    t1 = time.perf_counter()
    eng.scalars_async(res[t % 2].numpy(), t % 2)
    t2 = time.perf_counter()
    if t > 0: eng.scalars_wait((t - 1) % 2)
    t3 = time.perf_counter()
    print(f"{'row' if t % 2 == 0 else 'r1 '} issue {1e6*(t1-t0):.0f} async {1e6*(t2-t1):.0f} wait {1e6*(t3-t2):.0f}", file=sys.stderr)
eng.synchronize()
print(f"total {1e3*(time.perf_counter()-t00)/T:.3f} ms/step", file=sys.stderr)

"""Host-side cost per 5a step with host inputs (no per-step sync)."""
import sys, time
from pathlib import Path
import numpy as np
import torch
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa
from paper_2605_24514_b200 import BatchedSvdEngine  # noqa
dev = torch.device("cuda", 0)
T = 64
a0, rows, ii, jj, dd = bench.make_inputs(torch, dev, list(range(4096)), n_events=T)
eng = BatchedSvdEngine(a0, 32, m_cap=1024 + T, k_cap=32)
hr = torch.empty(rows.shape, dtype=torch.float64, pin_memory=True); hr.copy_(rows); hr = hr.numpy()
hi = ii.cpu().numpy(); hj = jj.cpu().numpy(); hd = dd.cpu().numpy()
eng.synchronize()
for name, fn in (("row host", lambda t: eng.row_append(hr[t])), ("row dev", lambda t: eng.row_append(rows[t])),
                 ("r1 host", lambda t: eng.rank_one_update(hi[t], hj[t], hd[t])),
                 ("r1 dev", lambda t: eng.rank_one_update(ii[t], jj[t], dd[t]))):
    tt = 0.0
    for t in range(8):
        eng.synchronize()
        t0 = time.perf_counter(); fn(t); t1 = time.perf_counter()
        tt += t1 - t0
    eng.synchronize()
    print(f"{name}: host issue {tt / 8 * 1e6:.0f} us")
x = np.ascontiguousarray(hr[0])
from paper_2605_24514_b200 import _lib
import ctypes
t0 = time.perf_counter()
for _ in range(20):
    np.isfinite(x).all()
print(f"numpy isfinite 8MB: {(time.perf_counter() - t0) / 20 * 1e6:.0f} us")
pg = np.ascontiguousarray(hr.copy())  # pageable copy
tt = 0.0
for t in range(8):
    eng.synchronize()
    t0 = time.perf_counter(); eng.row_append(pg[t]); tt += time.perf_counter() - t0
print(f"row pageable: host issue {tt / 8 * 1e6:.0f} us")
# raw H2D timings
d = torch.empty(hr[0].shape, dtype=torch.float64, device=dev)
src_p = torch.from_numpy(hr[0])
print("pinned?", src_p.is_pinned())
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(8):
    d.copy_(src_p, non_blocking=True)
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"torch H2D 8MB pinned: issue {(t1 - t0) / 8 * 1e6:.0f} us, total {(t2 - t0) / 8 * 1e6:.0f} us")
lib = _lib.load()
import ctypes
x = hr[0:1].reshape(1, -1) if hr.ndim == 2 else hr[0]
t0 = time.perf_counter()
for _ in range(8):
    eng.synchronize()
t1 = time.perf_counter()
print(f"sync cost {(t1 - t0) / 8 * 1e6:.0f} us")

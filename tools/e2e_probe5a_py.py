import sys, time
from pathlib import Path
import numpy as np
import torch
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa
from paper_2605_24514_b200 import BatchedSvdEngine, _lib  # noqa
from paper_2605_24514_b200.engine import _event_array  # noqa
dev = torch.device("cuda", 0)
T = 16
a0, rows, ii, jj, dd = bench.make_inputs(torch, dev, list(range(4096)), n_events=T)
eng = BatchedSvdEngine(a0, 32, m_cap=1024 + T, k_cap=32)
hr = torch.empty(rows.shape, dtype=torch.float64, pin_memory=True); hr.copy_(rows); hr = hr.numpy()
eng.synchronize()
for t in range(6):
    eng.synchronize()
    t0 = time.perf_counter()
    sh = eng._h.shape()
    t1 = time.perf_counter()
    src, d = _event_array(hr[t], (4096, 256), "row")
    t2 = time.perf_counter()
    rc = eng._h.lib.isvd_engine_row_append(eng._h.h, _lib.vptr(src), int(d))
    t3 = time.perf_counter()
    print(f"shape {1e6*(t1-t0):.0f} us, event_array {1e6*(t2-t1):.0f} us, C call {1e6*(t3-t2):.0f} us")

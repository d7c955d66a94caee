import sys, time
from pathlib import Path
import numpy as np
import torch
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa
from paper_2605_24514_b200 import BatchedSvdEngine, _lib  # noqa

m = 1 << 18
dev = torch.device("cuda", 0)
a0, rows = bench.make_inputs_5b(torch, dev, m=m)
eng = BatchedSvdEngine(a0, 128, m_cap=m + 300, k_cap=128)
h = torch.empty(rows.shape, dtype=torch.float64, pin_memory=True); h.copy_(rows); hr = h.numpy()
print("pinned", h.is_pinned())
pageable = rows.cpu().numpy().copy()
lib = _lib.load()
eng.synchronize()
def probe(name, get):
    ta = tb = 0.0
    for t in range(16):
        x = get(t)
        t0 = time.perf_counter()
        _lib.check(lib.isvd_engine_row_append(eng._h.h, _lib.vptr(x), int(torch.is_tensor(x))))
        t1 = time.perf_counter()
        eng.synchronize()
        t2 = time.perf_counter()
        if t >= 4:
            ta += t1 - t0; tb += t2 - t1
    print(f"{name}: issue {ta / 12 * 1e6:.1f} us wait {tb / 12 * 1e6:.1f} us")
probe("device", lambda t: rows[t:t + 1])
probe("pinned", lambda t: hr[t:t + 1])
probe("pageable", lambda t: pageable[t:t + 1])
probe("device", lambda t: rows[t:t + 1])
probe("pinned", lambda t: hr[t:t + 1])

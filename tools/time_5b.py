"""Config 5b (4,194,304 x 1024, k = 128, 256 row appends) timing breakdown."""
import ctypes
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2605_24514_b200 import BatchedSvdEngine, _lib  # noqa

m = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 22
n, k, T = 1024, 128, 256
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(5)
y = torch.randn(n, k, dtype=torch.float64, device=dev, generator=g)
a0 = torch.empty(m, n, dtype=torch.float64, device=dev)
step = 1 << 18
for c in range(0, m, step):
    s = min(step, m - c)
    x = torch.randn(s, k, dtype=torch.float64, device=dev, generator=g)
    a0[c:c + s] = x @ y.T + 1e-3 * torch.randn(s, n, dtype=torch.float64, device=dev, generator=g)
rows = torch.randn(T, k, dtype=torch.float64, device=dev, generator=g) @ y.T
torch.cuda.synchronize()
t0 = time.perf_counter()
eng = BatchedSvdEngine(a0.view(1, m, n), k, m_cap=m + T + 1, k_cap=k)
eng.synchronize()
print(f"init {time.perf_counter() - t0:.3f} s")
del a0
torch.cuda.empty_cache()
lib = _lib.load()
print("lazy window", lib.isvd_engine_lazy_window(eng._h.h))
i64p = ctypes.POINTER(ctypes.c_int64)
stream = torch.cuda.ExternalStream(eng.cuda_stream, device=dev)
for t in range(3):
    eng.row_append(rows[t:t + 1])
eng.flush()
eng.snapshot()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(stream)
for t in range(3, T):
    eng.row_append(rows[t:t + 1])
e1.record(stream)
eng.flush()
e2 = torch.cuda.Event(enable_timing=True)
e2.record(stream)
torch.cuda.synchronize()
ticks_ms = e0.elapsed_time(e1)
flush_ms = e1.elapsed_time(e2)
print(f"{T - 3} ticks {ticks_ms:.3f} ms ({ticks_ms / (T - 3) * 1e3:.1f} us/tick), final flush {flush_ms:.3f} ms,"
      f" updates/s {(T - 3) / ((ticks_ms + flush_ms) / 1e3):.0f}")
eng.restore()
_lib.check(lib.isvd_engine_set_timing(eng._h.h, 1))
for t in range(3, T):
    eng.row_append(rows[t:t + 1])
eng.flush()
ph = np.zeros(10)
nt = np.zeros(3, dtype=np.int64)
_lib.check(lib.isvd_engine_phase_times(eng._h.h, _lib.dptr(ph), nt.ctypes.data_as(i64p)))
print("per row tick ms: project %.4f core %.4f rotate %.4f install %.4f" % tuple(ph[:4] / max(1, nt[0])))
print(f"flushes {nt[2]} flush ms {ph[8]:.3f} bytes {ph[9] / 1e9:.2f} GB -> {ph[9] / (ph[8] / 1e3) / 1e9 if ph[8] else 0:.0f} GB/s,"
      f" {2.0 * m * k * k / (ph[8] / 1e3) / 1e12 if ph[8] else 0:.2f} TF/s")

"""Phase cycles of the column-split rotation (rotate_nsplit_kernel) on config
5b's per-tick W / V job (trace build, temporary K1_MARK marks)."""
import ctypes as C
import sys
from pathlib import Path
import numpy as np
import torch
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2605_24514_b200 import BatchedSvdEngine, _lib  # noqa
m = 1 << 18
n, k, T = 1024, 128, 40
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(5)
y = torch.randn(n, k, dtype=torch.float64, device=dev, generator=g)
x = torch.randn(m, k, dtype=torch.float64, device=dev, generator=g)
a0 = x @ y.T + 1e-3 * torch.randn(m, n, dtype=torch.float64, device=dev, generator=g)
rows = torch.randn(T, k, dtype=torch.float64, device=dev, generator=g) @ y.T
eng = BatchedSvdEngine(a0.view(1, m, n), k, m_cap=m + T + 1, k_cap=k)
del a0, x
lib = _lib.load()
for t in range(T):
    eng.row_append(rows[t].view(1, n))
eng.synchronize()
nb = 96
buf = (C.c_int64 * (nb * 10))()
_lib.check(lib.isvd_debug_trace(buf, -nb))
tr = np.array(buf, dtype=np.int64).reshape(nb, 10)[:, :5]
tr = tr[tr[:, 0] != 0]
d = np.diff(tr, axis=1).astype(np.float64)
print("CTAs traced", len(tr), "start spread", int(tr[:, 0].max() - tr[:, 0].min()), "end-to-end", int(tr[:, 4].max() - tr[:, 0].min()))
for i, nm in enumerate(["init+tma issue+zf", "first load issue", "tma wait", "groups"]):
    print(f"{nm:20s} median {np.median(d[:, i]):8.0f} max {d[:, i].max():8.0f}")

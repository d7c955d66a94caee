"""Phase cycles of the wide (cluster) secular solver on config 5b's 129-core
(library built with -DISVD_R1_TRACE):
  ISVD_NVCC_FLAGS=-DISVD_R1_TRACE python tools/trace_5b.py [m]"""
import ctypes as C
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2605_24514_b200 import BatchedSvdEngine, _lib  # noqa

m = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 18
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
names = ["setup", "csync", "roots", "csync", "loewner/pos", "csync", "vectors", "csync"]
acc = []
for t in range(T):
    eng.row_append(rows[t].view(1, n))
    eng.synchronize()
    buf = (C.c_int64 * 10)()
    _lib.check(lib.isvd_debug_trace(buf, 1))
    tr = np.array(buf, dtype=np.int64)[:9]
    if t >= 8 and tr[0] != 0:
        acc.append(np.diff(tr))
acc = np.array(acc, dtype=np.float64)
print(f"ticks traced: {len(acc)}")
for i, nm in enumerate(names):
    print(f"{nm:12s} median {np.median(acc[:, i]):8.0f}  max {acc[:, i].max():8.0f}  (SM cycles)")
print(f"{'total':12s} median {np.median(acc.sum(axis=1)):8.0f}")

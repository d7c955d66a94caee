"""Time isvd_core_svd on 4096 rank-1-shaped cores (diag(s) + delta a b^T)."""
import sys
from pathlib import Path
import numpy as np
import torch
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2605_24514_b200 import _lib  # noqa

lib = _lib.load()
B, s = 4096, 32
rng = np.random.default_rng(0)
sig = np.sort(rng.uniform(100, 900, size=(B, s)), axis=1)[:, ::-1]
a = rng.standard_normal((B, s)) * 0.03
b = rng.standard_normal((B, s)) * 0.06
cores = np.zeros((B, s, s))
for i in range(B):
    cores[i] = np.diag(sig[i]) + 0.01 * np.outer(a[i], b[i])
d = torch.tensor(cores, device="cuda")
u, vt = torch.empty_like(d), torch.empty_like(d)
sv = torch.empty((B, s), dtype=torch.float64, device="cuda")
for rep in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    _lib.check(lib.isvd_core_svd(B, s, d.data_ptr(), u.data_ptr(), sv.data_ptr(), vt.data_ptr(), None))
    e1.record()
    torch.cuda.synchronize()
    print("core_svd 4096 x 32:", e0.elapsed_time(e1), "ms")
# random dense cores for comparison
d2 = torch.randn((B, s, s), dtype=torch.float64, device="cuda")
for rep in range(2):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    _lib.check(lib.isvd_core_svd(B, s, d2.data_ptr(), u.data_ptr(), sv.data_ptr(), vt.data_ptr(), None))
    e1.record()
    torch.cuda.synchronize()
    print("core_svd random 4096 x 32:", e0.elapsed_time(e1), "ms")

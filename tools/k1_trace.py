"""Per-stream phase latencies of the projection kernel K1 (needs a library
built with -DISVD_R1_TRACE):

  ISVD_NVCC_FLAGS=-DISVD_R1_TRACE python tools/k1_trace.py [streams] [groups]

Runs config-5a-shaped ticks and prints, over the streams of the last row
append, the SM-clock cycles between consecutive marks of
project_append_kernel (median / p90 / p99 / max)."""
import ctypes as C
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2605_24514_b200 import BatchedSvdEngine, _lib  # noqa

B = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
m, n, k, r = 1024, 256, 32, 32
g = torch.Generator(device="cuda").manual_seed(0)
dev = torch.device("cuda")
x = torch.randn(B, m, r, device=dev, dtype=torch.float64, generator=g)
y = torch.randn(B, n, r, device=dev, dtype=torch.float64, generator=g)
a0 = torch.bmm(x, y.transpose(1, 2)) + 0.05 * torch.randn(B, m, n, device=dev, dtype=torch.float64, generator=g)
eng = BatchedSvdEngine(a0, k)
if len(sys.argv) > 2:
    _lib.check(_lib.load().isvd_engine_set_groups(eng._h.h, int(sys.argv[2])))
del a0, x
NT = int(sys.argv[3]) if len(sys.argv) > 3 else 47  # last tick is row append number 24 (nz = 7)
for t in range(NT):
    if t % 2 == 0:
        l = torch.randn(B, 1, r, device=dev, dtype=torch.float64, generator=g)
        row = torch.bmm(l, y.transpose(1, 2)).squeeze(1) + 0.05 * torch.randn(B, n, device=dev, dtype=torch.float64, generator=g)
        eng.row_append(row)
    else:
        mm = eng.shape[0]
        ii = torch.randint(0, mm, (B,), device=dev, generator=g)
        jj = torch.randint(0, n, (B,), device=dev, generator=g)
        dd = 0.01 * torch.randn(B, device=dev, dtype=torch.float64, generator=g)
        eng.rank_one_update(ii, jj, dd)
eng.synchronize()
lib = _lib.load()
nb = min(B, 4096)
buf = (C.c_int64 * (nb * 10))()
_lib.check(lib.isvd_debug_trace(buf, -nb))
tr = np.array(buf, dtype=np.int64).reshape(nb, 10)
tr = tr[tr[:, 0] != 0][:, :9]
names = ["setup/x/Z", "tma wait", "pass1", "G^T p", "G pc", "pass2", "rho sum", "core out"]
d = np.diff(tr, axis=1).astype(np.float64)
print(f"streams traced: {len(tr)}")
print(f"{'phase':10s} {'median':>8s} {'p90':>8s} {'p99':>8s} {'max':>8s}  (SM cycles)")
for i, nm in enumerate(names):
    v = d[:, i]
    print(f"{nm:10s} {np.median(v):8.0f} {np.percentile(v, 90):8.0f} {np.percentile(v, 99):8.0f} {v.max():8.0f}")
tot = (tr[:, 8] - tr[:, 0]).astype(np.float64)
print(f"{'total':10s} {np.median(tot):8.0f} {np.percentile(tot, 90):8.0f} {np.percentile(tot, 99):8.0f} {tot.max():8.0f}")

"""Per-core phase latencies of the CTA-per-core rank-1 kernel (needs a
library built with -DISVD_R1_TRACE):

  ISVD_NVCC_FLAGS=-DISVD_R1_TRACE python -m paper_2605_24514_b200.build --force
  python tools/r1_trace.py [streams]

Runs config-5a-shaped ticks (1024 x 256, rank 32 + N(0, 0.05^2), k = 32,
alternating row append / rank-1 on device inputs) and prints, over the cores
of the last rank-1 launch, the SM-clock cycles spent between consecutive
phase marks (median / p90 / p99 / max)."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2605_24514_b200 import BatchedSvdEngine, _lib  # noqa
import ctypes as C  # noqa

B = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
ARROW = "--arrow" in sys.argv  # trace the append-core kernel (last tick a row append)
m, n, k, r = 1024, 256, 32, 32
g = torch.Generator(device="cuda").manual_seed(0)
dev = torch.device("cuda")
x = torch.randn(B, m, r, device=dev, dtype=torch.float64, generator=g)
y = torch.randn(B, n, r, device=dev, dtype=torch.float64, generator=g)
a0 = torch.bmm(x, y.transpose(1, 2)) + 0.05 * torch.randn(B, m, n, device=dev, dtype=torch.float64, generator=g)
eng = BatchedSvdEngine(a0, k)
del a0, x
for t in range(41 if ARROW else 40):
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
cnt = (C.c_int64 * 8)()
lib.isvd_debug_counters(cnt, 0)
if cnt[2]:
    print(f"arrow roots {cnt[2]}, iterations per root {cnt[3] / cnt[2]:.2f}")
nb = min(B, 4096)
buf = (C.c_int64 * (nb * 10))()
_lib.check(lib.isvd_debug_trace(buf, nb))
tr = np.array(buf, dtype=np.int64).reshape(nb, 10)
tr = tr[tr[:, 0] != 0]
names = (["load/sort", "deflation", "roots", "loewner/pos", "vectors", "install", "epilogue"]
         if ARROW else ["gather", "gate", "step1", "G1", "dense", "sweep", "final", "UkVk", "epilogue"])
last = 7 if ARROW else 9
tr = tr[:, :last + 1]
d = np.diff(tr, axis=1).astype(np.float64)
print(f"cores traced: {len(tr)}")
print(f"{'phase':10s} {'median':>8s} {'p90':>8s} {'p99':>8s} {'max':>8s}  (SM cycles)")
for i, nm in enumerate(names):
    v = d[:, i]
    print(f"{nm:10s} {np.median(v):8.0f} {np.percentile(v, 90):8.0f} {np.percentile(v, 99):8.0f} {v.max():8.0f}")
tot = (tr[:, last] - tr[:, 0]).astype(np.float64)
print(f"{'total':10s} {np.median(tot):8.0f} {np.percentile(tot, 90):8.0f} {np.percentile(tot, 99):8.0f} {tot.max():8.0f}")

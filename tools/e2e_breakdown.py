"""Host-time breakdown of the 5a end-to-end loop (not a test): seconds spent
in each public call over N ticks with the bench's read-back lag."""
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2605_24514_b200 import BatchedSvdEngine, _lib  # noqa: E402

T, LAG = 256, int(sys.argv[1]) if len(sys.argv) > 1 else 2
G = int(sys.argv[2]) if len(sys.argv) > 2 else 4
dev = torch.device("cuda", 0)
a0, rows, ii, jj, dd = bench.make_inputs(torch, dev, list(range(4096)), n_events=T)
eng = BatchedSvdEngine(a0, 32, m_cap=1024 + T, k_cap=32)
_lib.check(_lib.load().isvd_engine_set_groups(eng._h.h, G))


def pinned(x):
    h = torch.empty(x.shape, dtype=x.dtype, pin_memory=True)
    h.copy_(x)
    return h.numpy()


hr, hi, hj, hd = (pinned(x) for x in (rows, ii, jj, dd))
res = torch.empty((8, 3 * 4096), dtype=torch.float64, pin_memory=True)
eng.snapshot()
for rep in range(2):
    eng.restore()
    eng.synchronize()
    acc = {"row": 0.0, "r1": 0.0, "async": 0.0, "wait": 0.0}
    t0 = time.perf_counter()
    for t in range(T):
        a = time.perf_counter()
        if t % 2 == 0:
            eng.row_append(hr[t // 2])
            acc["row"] += time.perf_counter() - a
        else:
            eng.rank_one_update(hi[t // 2], hj[t // 2], hd[t // 2])
            acc["r1"] += time.perf_counter() - a
        if LAG < 0:
            continue
        a = time.perf_counter()
        eng.scalars_async(res[t % 8].numpy(), t % 8)
        acc["async"] += time.perf_counter() - a
        a = time.perf_counter()
        if t >= LAG:
            eng.scalars_wait((t - LAG) % 8)
        acc["wait"] += time.perf_counter() - a
    for t in range(max(0, T - LAG), T if LAG >= 0 else 0):
        eng.scalars_wait(t % 8)
    eng.flush()
    eng.synchronize()
    tot = time.perf_counter() - t0
    print(f"lag {LAG} G {G}: {1e3 * tot / T:.4f} ms/tick; per tick us: " +
          ", ".join(f"{k} {1e6 * v / T:.1f}" for k, v in acc.items()))

"""Small driver for ncu: a 4096-stream cfg5a engine, a few ticks of each kind.
Usage: python tools/prof_ticks.py [n_ticks]"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402
from paper_2605_24514_b200 import BatchedSvdEngine  # noqa: E402

ticks = int(sys.argv[1]) if len(sys.argv) > 1 else 6
dev = torch.device("cuda", 0)
streams = list(range(4096))
a0, rows, ii, jj, dd = bench.make_inputs(torch, dev, streams, n_events=ticks)
eng = BatchedSvdEngine(a0, 32, m_cap=1024 + ticks + 1, k_cap=32)
for t in range(ticks):
    if t % 2 == 0:
        eng.row_append(rows[t // 2])
    else:
        eng.rank_one_update(ii[t // 2], jj[t // 2], dd[t // 2])
eng.flush()
torch.cuda.synchronize()
print("ok", eng.shape)

"""Secular-solver statistics on config-5b ticks (build with
ISVD_NVCC_FLAGS=-DISVD_ARROW_STATS)."""
import ctypes, sys
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
lib = _lib.load()
i64p = ctypes.POINTER(ctypes.c_int64)
dbg = np.zeros(8, dtype=np.int64)
eng.synchronize(); torch.cuda.synchronize()
lib.isvd_debug_counters(dbg.ctypes.data_as(i64p), 1)
for t in range(32):
    eng.row_append(rows[t:t + 1])
eng.synchronize(); torch.cuda.synchronize()
lib.isvd_debug_counters(dbg.ctypes.data_as(i64p), 1)
print("roots", dbg[2], "iters/root", dbg[3] / max(1, dbg[2]), "cores", dbg[4], "serial deflation", dbg[5])

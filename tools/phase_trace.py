"""Per-tick phase times of the cfg5a engine (serial, one group)."""
import ctypes, sys
from pathlib import Path
import numpy as np
import torch
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa
from paper_2605_24514_b200 import BatchedSvdEngine, _lib  # noqa

T = int(sys.argv[1]) if len(sys.argv) > 1 else 64
dev = torch.device("cuda", 0)
a0, rows, ii, jj, dd = bench.make_inputs(torch, dev, list(range(4096)), n_events=T)
eng = BatchedSvdEngine(a0, 32, m_cap=1024 + T + 1, k_cap=32)
lib = _lib.load()
i64p = ctypes.POINTER(ctypes.c_int64)
_lib.check(lib.isvd_engine_set_timing(eng._h.h, 1))
for t in range(T):
    if t % 2 == 0:
        eng.row_append(rows[t // 2])
    else:
        eng.rank_one_update(ii[t // 2], jj[t // 2], dd[t // 2])
    ph = np.zeros(10); nt = np.zeros(3, dtype=np.int64)
    dbg = np.zeros(8, dtype=np.int64)
    _lib.check(lib.isvd_engine_phase_times(eng._h.h, _lib.dptr(ph), nt.ctypes.data_as(i64p)))
    eng.synchronize(); torch.cuda.synchronize()
    _lib.check(lib.isvd_debug_counters(dbg.ctypes.data_as(i64p), 1))
    k = 0 if t % 2 == 0 else 4
    print(t, "row" if t % 2 == 0 else "r1 ", " ".join(f"{v:.3f}" for v in ph[k:k + 4]),
          f"sweeps={dbg[0] / max(1, dbg[1]):.2f}" if t % 2 else "")

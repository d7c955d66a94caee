"""Per-event latency of config-4-sized single-stream appends (20000 x 5000,
k = 64): synchronised row / column appends, with ISVD_HOST_PROF=1 for the
host sections."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2605_24514_b200 import SvdEngine, workloads  # noqa: E402

a0, ev, meta = workloads.cfg4(n_blocks=40)
e = SvdEngine(a0, int(sys.argv[1]) if len(sys.argv) > 1 else 64)
e.synchronize()
rows, cols = [], []
for t, x in enumerate(ev):
    t0 = time.perf_counter()
    if x[0] == "row":
        e.row_append(x[1])
    else:
        e.col_append(x[1])
    e.synchronize()
    (rows if x[0] == "row" else cols).append(time.perf_counter() - t0)
print(f"row median {1e6 * np.median(rows[10:]):.1f} us, col median {1e6 * np.median(cols[2:]):.1f} us")
del e

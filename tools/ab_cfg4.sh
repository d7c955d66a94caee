# A/B: config-4 single-stream event latency, round-1 library vs current
cd ab_old && python - 16 <<'PY'
import sys, time
sys.path.insert(0, '.')
sys.path.insert(1, '..')
import numpy as np
import paper_2605_24514_b200 as P
print("old pkg:", P.__file__)
from paper_2605_24514_b200 import SvdEngine, workloads
a0, ev, meta = workloads.cfg4(n_blocks=40)
e = SvdEngine(a0, int(sys.argv[1]) if len(sys.argv) > 1 else 64); e.synchronize()
rows, cols = [], []
for x in ev:
    t0 = time.perf_counter()
    (e.row_append if x[0] == "row" else e.col_append)(x[1]); e.synchronize()
    (rows if x[0] == "row" else cols).append(time.perf_counter() - t0)
print(f"OLD row median {1e6*np.median(rows[10:]):.1f} us, col median {1e6*np.median(cols[2:]):.1f} us")
PY
cd .. && python tools/cfg4_event_prof.py 16 2>&1 | tail -1

"""BASELINE config 4 at full size (20000 x 5000, rank 64, sigma_i = 0.9^i +
N(0, 0.01^2); 1000 x (5 row appends + 1 column append); adaptive rank
tau = 0.95, k <= 128; periodic refresh 500, metrics every 250) through the
package's run_stream.  Prints per-event update times and the trajectory."""
import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2605_24514_b200 import AdaptiveRankConfig, PolicyConfig, run_stream, workloads  # noqa
from paper_2605_24514_b200.linalg import orthonormality_defect  # noqa

blocks = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
t0 = time.perf_counter()
a0, events, meta = workloads.cfg4(n_blocks=blocks)
print(f"generated in {time.perf_counter() - t0:.1f} s", flush=True)
p = meta["policy"]
pol = PolicyConfig(kind="periodic", period=p["period"], adaptive=AdaptiveRankConfig(**p["adaptive"]))
t0 = time.perf_counter()
recs, eng = run_stream(a0, workloads.to_stream_events(events), meta["k"], pol,
                       log_every=meta["log_every"], return_engine=True)
wall = time.perf_counter() - t0
ut = np.array([r.update_time for r in recs[1:]])
kinds = [e[0] for e in events]
row_t = np.median([u for u, k in zip(ut, kinds) if k == "row"])
col_t = np.median([u for u, k in zip(ut, kinds) if k == "col"])
f = eng.factors
out = {"events": len(events), "wall_s": wall, "init_s": recs[0].update_time,
       "median_row_update_ms": 1e3 * row_t, "median_col_update_ms": 1e3 * col_t,
       "refreshes": int(sum(r.refreshed for r in recs)), "final_shape": list(eng.shape),
       "final_rank": int(f.s.size), "ortho_u": orthonormality_defect(f.u),
       "ortho_v": orthonormality_defect(f.vt.T),
       "logged": [{"t": r.step, "ratio": r.frob_ratio, "evr": r.evr, "rank": r.rank, "refreshed": r.refreshed}
                  for r in recs if r.frob_ratio is not None][:40]}
print(json.dumps(out, indent=1))

import sys, time
sys.path.insert(0, '.')
import numpy as np
from paper_2605_24514_b200 import SvdEngine, workloads
a0, ev, meta = workloads.cfg1()
e = SvdEngine(a0, 10)
for x in ev[:50]: e.row_append(x[1])
e.synchronize()
t0 = time.perf_counter()
for x in ev[50:450]: e.row_append(x[1])
t1 = time.perf_counter(); e.synchronize()
print("cfg1 enqueue us", 1e6*(t1-t0)/400)
del e
a0, ev, meta = workloads.cfg2(n_events=450)
e = SvdEngine(a0, 20)
for x in ev[:50]: e.rank_one_update(x[1], x[2], x[3])
e.synchronize()
t0 = time.perf_counter()
for x in ev[50:450]: e.rank_one_update(x[1], x[2], x[3])
t1 = time.perf_counter(); e.synchronize()
print("cfg2 enqueue us", 1e6*(t1-t0)/400)
del e

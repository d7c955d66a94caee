import sys, time
from pathlib import Path
import numpy as np
import torch
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa
from paper_2605_24514_b200 import BatchedSvdEngine  # noqa
dev = torch.device("cuda", 0)
T = 64
a0, rows, ii, jj, dd = bench.make_inputs(torch, dev, list(range(4096)), n_events=T)
eng = BatchedSvdEngine(a0, 32, m_cap=1024 + 4 * T, k_cap=32)
import os
from paper_2605_24514_b200 import _lib
if os.environ.get("G"):
    _lib.check(_lib.load().isvd_engine_set_groups(eng._h.h, int(os.environ["G"])))
hr = torch.empty(rows.shape, dtype=torch.float64, pin_memory=True); hr.copy_(rows); hr = hr.numpy()
hi = torch.empty(ii.shape, dtype=torch.int64, pin_memory=True); hi.copy_(ii); hi = hi.numpy()
hj = torch.empty(jj.shape, dtype=torch.int64, pin_memory=True); hj.copy_(jj); hj = hj.numpy()
hd = torch.empty(dd.shape, dtype=torch.float64, pin_memory=True); hd.copy_(dd); hd = hd.numpy()
res = torch.empty((2, 3 * 4096), dtype=torch.float64, pin_memory=True)
eng.snapshot()
def loop(host, mode, hrow=None, hr1=None):
    hrow = host if hrow is None else hrow
    hr1 = host if hr1 is None else hr1
    eng.restore(); eng.synchronize()
    t0 = time.perf_counter()
    for t in range(T):
        if t % 2 == 0:
            eng.row_append(hr[t // 2] if hrow else rows[t // 2])
        else:
            if hr1: eng.rank_one_update(hi[t // 2], hj[t // 2], hd[t // 2])
            else: eng.rank_one_update(ii[t // 2], jj[t // 2], dd[t // 2])
        if mode == "lag":
            eng.scalars_async(res[t % 2].numpy(), t % 2)
            if t > 0: eng.scalars_wait((t - 1) % 2)
        elif mode == "sync":
            eng.scalars()
    eng.synchronize()
    return (time.perf_counter() - t0) / T * 1e3
for host in (False, True):
    for mode in ("none", "lag", "sync"):
        print(f"host={host} mode={mode}: {loop(host, mode):.3f} ms/step")
print(f"host rows only, lag: {loop(False, 'lag', True, False):.3f}")
print(f"host r1 only, lag: {loop(False, 'lag', False, True):.3f}")
eng.restore(); eng.synchronize()
ta = tb = tc = 0.0
for t in range(T):
    t0 = time.perf_counter()
    if t % 2 == 0:
        eng.row_append(hr[t // 2])
    else:
        eng.rank_one_update(ii[t // 2], jj[t // 2], dd[t // 2])
    t1 = time.perf_counter()
    eng.scalars_async(res[t % 2].numpy(), t % 2)
    t2 = time.perf_counter()
    if t > 0: eng.scalars_wait((t - 1) % 2)
    t3 = time.perf_counter()
    if t % 2 == 0 and t > 8:
        print(f"row step: issue {1e6*(t1-t0):.0f} async {1e6*(t2-t1):.0f} wait {1e6*(t3-t2):.0f}")
    if t % 2 == 1 and t > 8 and t < 16:
        print(f"r1 step: issue {1e6*(t1-t0):.0f} async {1e6*(t2-t1):.0f} wait {1e6*(t3-t2):.0f}")
print("---- gpu timeline (lag mode, host rows)")
eng.restore(); eng.synchronize()
st = torch.cuda.ExternalStream(eng.cuda_stream, device=dev)
evs = []
for t in range(24):
    e0 = torch.cuda.Event(enable_timing=True); e0.record(st)
    if t % 2 == 0:
        eng.row_append(hr[t // 2])
    else:
        eng.rank_one_update(ii[t // 2], jj[t // 2], dd[t // 2])
    e1 = torch.cuda.Event(enable_timing=True); e1.record(st)
    evs.append((e0, e1))
    eng.scalars_async(res[t % 2].numpy(), t % 2)
    if t > 0: eng.scalars_wait((t - 1) % 2)
eng.synchronize()
for t in range(12, 20):
    e0, e1 = evs[t]
    gap = evs[t - 1][1].elapsed_time(e0)
    print(f"step {t} {'row' if t % 2 == 0 else 'r1 '}: gpu {e0.elapsed_time(e1):.3f} ms, idle before {gap:.3f} ms")
import sys as _s; _s.exit(0)
print("---- device rows, concurrent 8MB H2D on a side stream during r1")
eng.restore(); eng.synchronize()
side = torch.cuda.Stream()
dst = torch.empty(hr[0].shape, dtype=torch.float64, device=dev)
src = torch.from_numpy(hr[0])
evs = []
for t in range(24):
    e0 = torch.cuda.Event(enable_timing=True); e0.record(st)
    if t % 2 == 0:
        eng.row_append(rows[t // 2])
    else:
        eng.rank_one_update(ii[t // 2], jj[t // 2], dd[t // 2])
        with torch.cuda.stream(side):
            dst.copy_(src, non_blocking=True)
    e1 = torch.cuda.Event(enable_timing=True); e1.record(st)
    evs.append((e0, e1))
eng.synchronize(); torch.cuda.synchronize()
for t in range(12, 18):
    e0, e1 = evs[t]
    print(f"step {t} {'row' if t % 2 == 0 else 'r1 '}: gpu {e0.elapsed_time(e1):.3f} ms")

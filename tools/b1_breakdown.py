"""Where the single-stream (B = 1) event latency goes, configs 1-3:
  * host enqueue: the API call without a synchronisation (Python + libisvd
    host work + launches), averaged over a burst of events;
  * device+sync: per event with a synchronisation after it (the
    update_time the stream loop records, stream.py:284-289);
  * launches per event (isvd_launch_count).
  python tools/b1_breakdown.py
"""
import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2605_24514_b200 import SvdEngine, _lib, workloads  # noqa: E402


def apply(e, ev):
    if ev[0] == "row":
        e.row_append(ev[1])
    elif ev[0] == "col":
        e.col_append(ev[1])
    else:
        e.rank_one_update(ev[1], ev[2], ev[3])


def run(name, a0, events, k, n=400):
    lib = _lib.load()
    evs = events[:n]
    e = SvdEngine(a0, k)
    for ev in evs[:16]:
        apply(e, ev)
    e.synchronize()
    e = SvdEngine(a0, k)
    e.synchronize()
    l0 = lib.isvd_launch_count()
    t0 = time.perf_counter()
    for ev in evs:
        apply(e, ev)
    t1 = time.perf_counter()
    e.synchronize()
    t2 = time.perf_counter()
    launches = (lib.isvd_launch_count() - l0) / len(evs)
    e = SvdEngine(a0, k)
    e.synchronize()
    per = []
    for ev in evs:
        s0 = time.perf_counter()
        apply(e, ev)
        e.synchronize()
        per.append(time.perf_counter() - s0)
    return {"events": len(evs), "enqueue_us": 1e6 * (t1 - t0) / len(evs),
            "burst_total_us": 1e6 * (t2 - t0) / len(evs),
            "synced_median_us": 1e6 * float(np.median(per)), "launches_per_event": launches}


def main():
    out = {}
    a0, ev, meta = workloads.cfg1()
    out["cfg1_rows"] = run("cfg1", a0, ev, meta["k"])
    a0, ev, meta = workloads.cfg2(n_events=1000)
    out["cfg2_rank1"] = run("cfg2", a0, ev, meta["k"])
    a0, ev, meta = workloads.cfg3()
    out["cfg3_rows"] = run("cfg3", a0, ev, meta["k"])
    out["cfg1_host_split"] = host_split()
    print(json.dumps(out, indent=1))



def host_split(n=400):
    """cfg1 row appends: the Python API vs a direct C-ABI call (pageable and
    pinned payloads), enqueue cost per event without synchronisation."""
    import torch

    lib = _lib.load()
    a0, ev, meta = workloads.cfg1()
    xs = np.stack([e[1] for e in ev[:n]])
    pinned = torch.empty(xs.shape, dtype=torch.float64, pin_memory=True)
    pinned.copy_(torch.from_numpy(xs))
    pn = pinned.numpy()
    out = {}
    for name, mode in (("python_api", 0), ("cabi_pageable", 1), ("cabi_pinned", 2)):
        e = SvdEngine(a0, meta["k"])
        e.synchronize()
        h = e._h.h
        t0 = time.perf_counter()
        for t in range(n):
            if mode == 0:
                e.row_append(xs[t])
            else:
                src = xs[t] if mode == 1 else pn[t]
                _lib.check(lib.isvd_engine_row_append(h, src.ctypes.data, 0))
        t1 = time.perf_counter()
        e.synchronize()
        out[name + "_enqueue_us"] = 1e6 * (t1 - t0) / n
    return out


if __name__ == "__main__":
    main()

"""Per-event update latency for BASELINE configs 1-3 (and config 4 on a
reduced panel): the GPU engine (each event synchronised, so the time is the
full device latency of one update) next to the CPU restatement of the
reference engine (oracle/, numpy + LAPACK on the host) on the same seeded
events -- SURVEY.md 8(d): "report reference per-tick update_time medians next
to the GPU per-tick latency".  Also checks the final factors agree (sigma
relative, sine angle).  Writes one JSON object to stdout.

  python tools/latency_cfgs.py [n_cpu_events]
"""
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from oracle import OracleEngine, sine_angle_max  # noqa: E402  (checker / CPU baseline only)
from paper_2605_24514_b200 import SvdEngine, workloads  # noqa: E402


def apply(e, ev):
    if ev[0] == "row":
        e.row_append(ev[1])
    elif ev[0] == "col":
        e.col_append(ev[1])
    else:
        e.rank_one_update(ev[1], ev[2], ev[3])


VDEFER = None  # engine default unless set (tools/latency_cfgs.py n_cpu vdefer_mode)


def run(name, a0, events, k, n_cpu):
    gpu = SvdEngine(a0, k)
    gpu.synchronize()
    times = {}
    for ev in events[:8]:  # warm-up (first-launch costs), then restart
        apply(gpu, ev)
    gpu = SvdEngine(a0, k)
    if VDEFER is not None:
        gpu.set_vdefer(VDEFER)
    gpu.synchronize()
    for ev in events:
        t0 = time.perf_counter()
        apply(gpu, ev)
        gpu.synchronize()
        times.setdefault(ev[0], []).append(time.perf_counter() - t0)
    cpu = OracleEngine(a0, k)
    ctimes = {}
    for ev in events[:n_cpu]:
        t0 = time.perf_counter()
        apply(cpu, ev)
        ctimes.setdefault(ev[0], []).append(time.perf_counter() - t0)
    out = {"events": len(events), "k": k, "shape0": list(a0.shape)}
    for kind in times:
        g = 1e6 * float(np.median(times[kind]))
        c = 1e6 * float(np.median(ctimes.get(kind, [np.nan])))
        out[kind] = {"gpu_median_us": g, "cpu_median_us": c, "cpu_over_gpu": c / g,
                     "gpu_events": len(times[kind]), "cpu_events": len(ctimes.get(kind, []))}
    # parity of the full-length GPU run against the CPU restatement when the
    # CPU also ran the whole stream
    if n_cpu >= len(events):
        fg, fc = gpu.factors, cpu.factors
        out["sigma_rel"] = float(np.max(np.abs(fg.s - fc.s) / np.maximum(fc.s, 1e-300)))
        out["angle_u"] = float(sine_angle_max(fg.u, fc.u))
        out["angle_v"] = float(sine_angle_max(fg.vt.T, fc.vt.T))
    return out


def main():
    global VDEFER
    n_cpu = int(sys.argv[1]) if len(sys.argv) > 1 else 10**9
    if len(sys.argv) > 2:
        VDEFER = int(sys.argv[2])
    res = {"note": "per-event latency (GPU: synchronised after every event; CPU: oracle/ "
                   "numpy restatement of the reference engine, LAPACK core SVD), "
                   "metrics and refreshes excluded"}
    a0, ev, meta = workloads.cfg1()
    res["cfg1_rows"] = run("cfg1", a0, ev, meta["k"], n_cpu)
    a0, ev, meta = workloads.cfg2(n_events=2000)
    res["cfg2_rank1"] = run("cfg2", a0, ev, meta["k"], n_cpu)
    a0, ev, meta = workloads.cfg3()
    res["cfg3_rows"] = run("cfg3", a0, ev, meta["k"], n_cpu)
    a0, ev, meta = workloads.cfg4(m=4000, n=1000, n_blocks=50)
    res["cfg4_small_mixed"] = run("cfg4", a0, ev, meta["k"], n_cpu)
    print(json.dumps(res))


if __name__ == "__main__":
    main()

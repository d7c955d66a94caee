"""Benchmark: BASELINE config 5a -- batched incremental-SVD streams on B200.

Workload (BASELINE.json configs[4] part a, the config the headline metric
"iSVD updates/sec (k=32)" is quoted on): 4096 independent streams, each a
1024 x 256 rank-32 Gaussian product plus N(0, 0.05^2) noise, k = 32; 1024
events per stream alternating row append and rank-1 update (delta ~
N(0, 0.01)).  One step = one tick = one event applied to every stream.
Streams are sharded across ranks (strong scaling: the 4096 streams are split
over N GPUs, no data-path collective).

`value`   updates/s with inputs resident in HBM (device-event timing on the
          engine's stream, max over ranks).
`e2e`     the same through the public API with pinned HOST event buffers:
          host validation + H2D copy + kernels + D2H read of the step's
          result (per-stream sq_norm, residual and input norm) every step;
          the host waits for step t's result after issuing step t+1.
`roofline` the dominant kernel by time against its binding resource (FP64
          tensor peak for the core kernels, HBM for K1 / rotations):
          algorithmic flops or bytes / its measured duration (CUDA events on
          the engine stream).
`rotation` BASELINE's "basis-rotation HBM GB/s": the deferred U flush and the
          V materialisation (algorithmic bytes / measured time vs HBM peak).

`--impl reference` times the reference algorithm's CPU implementation (the
numpy restatement in oracle/, all host cores) on a bounded sample of the
same workload, printing the same JSON line with "impl": "reference".
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

M0, N0, RANK, K = 1024, 256, 32, 32
TOTAL_STREAMS = 4096
EVENTS = 1024
# e2e host loop: results are read back E2E_LAG steps behind their issue
E2E_LAG, RES_SLOTS = 2, 4
METRIC = "iSVD updates/sec (k=32)"
UNIT = "updates/s"
# BASELINE configs[4] part b: one tall matrix, k = 128, 256 row appends
M5B, N5B, RANK5B, K5B, T5B = 1 << 22, 1024, 128, 128, 256
DMMA_PEAK_TFS = 37.06  # measured FP64 DMMA.8x8x4 peak, profiles/r01_fp64_peaks.txt


def _ncu_summary():
    """Per-kernel ncu --set full figures committed under profiles/ (for the
    roofline `traffic` field); {} when absent."""
    for p in sorted((ROOT / "profiles").glob("r*_tick_ncu_summary.json"), reverse=True):
        try:
            return json.loads(p.read_text()), p.name
        except Exception:
            continue
    return {}, None


def _peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d.get("hbm_gbs", 6650.0)), "measured"
    return 6650.0, "fallback"


# ------------------------------------------------------------ reference arm
def _ref_worker(args):
    """One CPU worker: its streams through the oracle engine (numpy/LAPACK),
    single BLAS thread; returns (updates, seconds excluding init)."""
    seed, streams, n_events = args
    os.environ["OMP_NUM_THREADS"] = "1"
    from oracle import OracleEngine
    from paper_2605_24514_b200 import workloads

    engines, evs = [], []
    for b in streams:
        a0, ev = workloads.cfg5a_stream(seed, b, n_events=n_events)
        engines.append(OracleEngine(a0, K))
        evs.append(ev)
    t0 = time.perf_counter()
    for t in range(n_events):
        for e, ev in zip(engines, evs):
            x = ev[t]
            if x[0] == "row":
                e.row_append(x[1])
            else:
                e.rank_one_update(x[1], x[2], x[3])
    return len(streams) * n_events, time.perf_counter() - t0


def cpu_reference(n_streams: int, n_events: int, seed: int = 0):
    """Aggregate updates/s of the CPU reference implementation over all host
    cores (multiprocessing, one BLAS thread per worker)."""
    import multiprocessing as mp

    cores = len(os.sched_getaffinity(0))
    workers = min(cores, n_streams)
    chunks = [list(range(w, n_streams, workers)) for w in range(workers)]
    env_before = os.environ.get("OMP_NUM_THREADS")
    os.environ["OMP_NUM_THREADS"] = "1"
    ctx = mp.get_context("spawn")
    with ctx.Pool(workers) as pool:
        res = pool.map(_ref_worker, [(seed, c, n_events) for c in chunks])
    if env_before is None:
        os.environ.pop("OMP_NUM_THREADS", None)
    else:
        os.environ["OMP_NUM_THREADS"] = env_before
    updates = sum(r[0] for r in res)
    secs = max(r[1] for r in res)
    return updates / secs, workers, updates, secs


def cpu_reference_5b(ticks: int = 3, seed: int = 0):
    """The reference's row-append kernel (oracle/ restatement of
    _kernels_py.row_append, numpy/BLAS on all host cores) on a full-size
    config-5b factor set: U 4,194,304 x 128, Vt 128 x 1024.  Per SURVEY 8(d)
    the engine path's 34 GB vstack and infeasible init SVD are excluded."""
    from oracle import kernel_row_append

    rng = np.random.default_rng([seed, 55])
    # ~orthonormal columns; a tiled block keeps the 4.3 GB setup to a memcpy
    u = np.tile(rng.standard_normal((1 << 16, K5B)) / math.sqrt(M5B), (M5B >> 16, 1))
    vt = np.linalg.qr(rng.standard_normal((N5B, K5B)))[0].T.copy()
    s_ = np.sort(rng.uniform(1.0, 100.0, K5B))[::-1].copy()
    xs = rng.standard_normal((ticks, K5B)) @ vt
    t0 = time.perf_counter()
    for t in range(ticks):
        u2, s2, vt2, _ = kernel_row_append(u, s_, vt, xs[t], 1e-10, K5B)
        u = u2[:M5B]  # keep the height fixed so every sample tick costs the same
        s_, vt = s2, vt2
    secs = time.perf_counter() - t0
    return ticks / secs, len(os.sched_getaffinity(0)), ticks, secs


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    # bounded sample: 64 streams; each "step" = one event on every sampled stream
    n_streams = 64
    steps = max(1, args.steps)
    value, cores, updates, secs = cpu_reference(n_streams, steps + args.warmup)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * secs / (steps + args.warmup), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "cfg5a_batched_streams", "streams_sampled": n_streams,
                   "m0": M0, "n": N0, "k": K, "events_per_stream": steps + args.warmup},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": f"{n_streams} cfg5a streams x {steps + args.warmup} events "
                                   f"(oracle/ numpy restatement, LAPACK core SVD, 1 BLAS thread "
                                   f"per worker, init excluded)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    if not args.no_k128:
        v5, c5, t5, s5 = cpu_reference_5b()
        line["k128"] = {"metric": "iSVD updates/sec (k=128)", "value": v5, "unit": UNIT,
                        "config": {"workload": "cfg5b_tall", "m": M5B, "n": N5B, "k": K5B},
                        "cpu_baseline": {"value": v5, "unit": UNIT, "cores": c5, "kind": "port",
                                         "sample": f"{t5} full-size row appends through the "
                                                   "oracle row-append kernel (numpy/BLAS, all "
                                                   "host threads), engine vstack excluded"}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ GPU arm
class ClockSampler:
    def __init__(self, path):
        self.path = path
        self.proc = None

    def __enter__(self):
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={q}", "--format=csv",
                                          "-lms", "50"], stdout=self.f,
                                         stderr=subprocess.DEVNULL)
            time.sleep(0.5)  # let the sampler start before the timed region
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc:
            time.sleep(0.1)
            self.proc.terminate()
            self.proc.wait()
            self.f.close()

    def summary(self, gpu_index=0):
        try:
            lines = Path(self.path).read_text().strip().splitlines()[1:]
        except Exception:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9 or parts[0] != str(gpu_index):
                continue
            try:
                sm.append(float(parts[1].split()[0]))
                mx = float(parts[2].split()[0])
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def make_inputs(torch, dev, streams, seed=0, n_events=EVENTS):
    """Seeded device-side synthetic inputs for the local streams (torch
    Philox per stream id, so shards are independent of the world size)."""
    B = len(streams)
    a0 = torch.empty((B, M0, N0), dtype=torch.float64, device=dev)
    ys = torch.empty((B, N0, RANK), dtype=torch.float64, device=dev)
    g = torch.Generator(device=dev)
    for i, b in enumerate(streams):
        g.manual_seed(1_000_003 * seed + b)
        x = torch.randn((M0, RANK), dtype=torch.float64, device=dev, generator=g)
        y = torch.randn((N0, RANK), dtype=torch.float64, device=dev, generator=g)
        a0[i] = x @ y.T + 0.05 * torch.randn((M0, N0), dtype=torch.float64, device=dev, generator=g)
        ys[i] = y
    g.manual_seed(7_777_777 + seed * 131 + streams[0])
    nrow = (n_events + 1) // 2
    nr1 = n_events // 2
    rows = torch.empty((nrow, B, N0), dtype=torch.float64, device=dev)
    for t in range(nrow):
        l = torch.randn((B, RANK, 1), dtype=torch.float64, device=dev, generator=g)
        rows[t] = torch.bmm(ys, l).squeeze(-1) + 0.05 * torch.randn((B, N0), dtype=torch.float64,
                                                                    device=dev, generator=g)
    ii = torch.empty((nr1, B), dtype=torch.int64, device=dev)
    for t in range(nr1):
        m_now = M0 + t + 1  # rows appended before rank-1 tick 2t+1
        ii[t] = torch.randint(0, m_now, (B,), device=dev, generator=g)
    jj = torch.randint(0, N0, (nr1, B), device=dev, generator=g)
    dd = 0.01 * torch.randn((nr1, B), dtype=torch.float64, device=dev, generator=g)
    return a0, rows, ii, jj, dd


def rotation_bytes(B, m, n, r, keep, row_tick):
    """Algorithmic HBM bytes of one rotation launch (K3+K4 over B streams):
    U read m x r + written (m [+1]) x keep, V read n x r + written n x keep,
    plus the injected residual z (n) on row appends."""
    if row_tick:
        return 8 * B * (m * r + (m + 1) * keep + n * r + n * keep + n)
    return 8 * B * (m * r + m * keep + n * r + n * keep)


def tick_bytes(B, m, n, w, row_tick):
    """SURVEY.md 8(d) algorithmic bytes per update (whole tick)."""
    if row_tick:
        return 8 * B * (2 * m * w + 2 * n * w + 2 * n)
    return 8 * B * (2 * m * w + 2 * n * w + 2 * w + 2)


def _simulate_bytes(B, steps, window=32, vwin=8):
    """Algorithmic bytes of the per-tick kernels over `steps` ticks, following
    the engine's data flow: the deferred left basis (W =
    (32 + b) x 32 rotated in place, flushed every `window` appended rows) and
    the deferred right basis V_eff = [V | Z^T] G (a rank-1 tick rotates G; a
    full-rank row tick projects through V, Z and G, writes its residual as the
    next Z column and grows G by a row; V is materialised every `vwin` row
    appends).  Returns (projection bytes, row-tick and rank-1-tick rotation
    bytes (moved inside the core kernels), V-materialisation bytes, SURVEY
    8(d) reference-algorithm bytes)."""
    proj_bytes = rot_row = rot_r1 = vflush_bytes = all_bytes = 0.0
    m, b_rows, active = M0, 0, False
    vpend, nz = False, 0
    for t in range(steps):
        row = t % 2 == 0
        all_bytes += tick_bytes(B, m, N0, K, row)
        g = (K + nz) * K if vpend else 0                      # rows of G x K
        if row:
            # V and Z read once, x read, A row + residual written, G read
            proj_bytes += 8.0 * B * (N0 * K + nz * N0 + N0 + 2 * N0 + g)
            vb = g + (K + nz + 1) * K                         # G read, grown G written
            if not vpend:
                vpend, nz = True, 0
            nz += 1
            if nz >= vwin:                                    # V <- [V | Z^T] G
                vflush_bytes += 8.0 * B * (N0 * K + nz * N0 + (K + nz) * K + N0 * K)
                vpend, nz = False, 0
            if not active:
                wb = (K + 1) * K                              # W = Uk copy
                active, b_rows = True, 1
            else:
                wb = (K + b_rows) * K + (K + b_rows + 1) * K
                b_rows += 1
            m += 1
            if b_rows >= window:
                active, b_rows = False, 0
        else:
            rot_r1 += 8.0 * B * (2 * K + 2 + nz)              # U/V row gathers (+ Z entries)
            vb = 2 * g if vpend else K * K                    # G <- G Vk, or Vk written as G
            vpend = True
            if not active:
                wb = K * K
                active, b_rows = True, 0
            else:
                wb = 2 * (K + b_rows) * K
        if row:
            rot_row += 8.0 * B * (vb + wb)
        else:
            rot_r1 += 8.0 * B * (vb + wb)
    return proj_bytes, rot_row, rot_r1, vflush_bytes, all_bytes


def _simulate_flops(B, steps, window=32, vwin=8, rank1_steps=2.0):
    """Algorithmic FP64 flops of the two core kernels over `steps` ticks,
    following the same data flow as _simulate_bytes:
    * rank-1 tick (rank1_fast_kernel): the core factorisation as the
      simultaneous Jacobi steps run it -- the first step from the structure
      of K (Gram and rotation O(k^2); Theta^2 is symmetric: k^3), each
      further step the symmetric 32 x 32 Gram (k^3) and G (J - I) (2 k^3) --
      plus the fused rotations of the deferred bases: W (rows_W x k) . Uk and
      G (rows_G x k) . Vk (2 rows k^2 each).  (Symmetric products are counted
      once: the model stays at or below what ncu counts as executed tensor
      flops, profiles/r*_tick_ncu_summary.json r1fast.tensor_fp64_ops.)
    * row tick (arrow): the secular solve is O(k^2) (counted as 40 (k+1)^2)
      plus the fused rotations [W 0; 0 1] . Q and [G 0; 0 1] . Vk (2 rows (k+1) k).
    Returns (rank-1 flops, row flops)."""
    k = K
    f_r1 = f_row = 0.0
    b_rows, active = 0, False
    vpend, nz = False, 0
    core = 1.0 * k ** 3 + 3.0 * k ** 3 * max(0.0, rank1_steps - 1.0)
    for t in range(steps):
        row = t % 2 == 0
        g_rows = (k + nz) if vpend else 0
        if row:
            w_rows = k + b_rows if active else 0
            f_row += B * (40.0 * (k + 1) ** 2 + 2.0 * (w_rows + 1) * (k + 1) * k
                          + 2.0 * (g_rows + 1) * (k + 1) * k)
            if not vpend:
                vpend, nz = True, 0
            nz += 1
            if nz >= vwin:
                vpend, nz = False, 0
            if not active:
                active, b_rows = True, 1
            else:
                b_rows += 1
            if b_rows >= window:
                active, b_rows = False, 0
        else:
            w_rows = k + b_rows if active else k
            f_r1 += B * (core + 2.0 * w_rows * k * k + 2.0 * g_rows * k * k)
            vpend = True
            if not active:
                active, b_rows = True, 0
    return f_r1, f_row


def make_inputs_5b(torch, dev, seed=0, m=M5B, row0=0, rows=None):
    """Config 5b: A0 = X Y^T (m x 1024, rank 128) + N(0, 1e-3^2), appended rows
    l.Y^T.  Generated on the device in 2^18-row chunks, each
    from its own seed, so a rank builds exactly its row block [row0, row0 +
    rows) and every world size sees the same matrix."""
    rows = m - row0 if rows is None else rows
    chunk = 1 << 18
    g = torch.Generator(device=dev).manual_seed(5_000_011 + seed)
    y = torch.randn((N5B, RANK5B), dtype=torch.float64, device=dev, generator=g)
    app = torch.randn((T5B, RANK5B), dtype=torch.float64, device=dev, generator=g) @ y.T
    a0 = torch.empty((1, rows, N5B), dtype=torch.float64, device=dev)
    for c0 in range(row0 // chunk * chunk, row0 + rows, chunk):
        g.manual_seed(5_100_000 + 1000 * seed + c0 // chunk)
        h = min(chunk, m - c0)
        x = torch.randn((h, RANK5B), dtype=torch.float64, device=dev, generator=g)
        blk = x @ y.T + 1e-3 * torch.randn((h, N5B), dtype=torch.float64, device=dev, generator=g)
        lo, hi = max(row0, c0), min(row0 + rows, c0 + h)
        a0[0, lo - row0:hi - row0] = blk[lo - c0:hi - c0]
        del x, blk
    return a0, app.contiguous()


def run_cfg5b(torch, dev, lib, warm, world=1, rank=0):
    """Config 5b leg (k = 128): value = row appends/s with the final flush
    (materialising U) inside the timed region, max over ranks; e2e through the
    public API with pinned host rows; roofline of the deferred U rotation
    (FP64 DMMA).  N > 1: U and A row-sharded over the ranks
    (ShardedSvdEngine, NCCL allreduce of the Grams at init)."""
    import ctypes

    from paper_2605_24514_b200 import BatchedSvdEngine
    from paper_2605_24514_b200.sharded import ShardedSvdEngine, shard_rows
    from paper_2605_24514_b200.sharding import max_over_ranks

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            import torch.distributed as dist
            dist.barrier()

    i64p = ctypes.POINTER(ctypes.c_int64)
    r0, ml = shard_rows(M5B, world, rank)
    a0, rows = make_inputs_5b(torch, dev, row0=r0, rows=ml)
    barrier()
    t0 = time.perf_counter()
    if world == 1:
        eng = BatchedSvdEngine(a0, K5B, m_cap=M5B + T5B + 1, k_cap=K5B)
    else:
        eng = ShardedSvdEngine(a0[0], K5B, m_global=M5B, row0=r0, rows_cap=ml + T5B + 1,
                               k_cap=K5B)
    eng.synchronize()
    init_s = time.perf_counter() - t0
    del a0
    torch.cuda.empty_cache()
    stream = torch.cuda.ExternalStream(eng.cuda_stream, device=dev)
    for t in range(warm):
        eng.row_append(rows[t:t + 1])
    eng.flush()
    eng.snapshot()
    steps = T5B - warm
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    l0 = lib.isvd_launch_count()
    e0.record(stream)
    for t in range(warm, T5B):
        eng.row_append(rows[t:t + 1])
    eng.flush()
    e1.record(stream)
    barrier()
    launches = lib.isvd_launch_count() - l0
    ms = max_over_ranks(e0.elapsed_time(e1), device=dev)
    du, dv = (np.ravel(v)[0] for v in eng.ortho_defect())
    # per-phase breakdown of the same ticks
    eng.restore()
    lib.isvd_engine_set_timing(eng._h.h, 1)
    for t in range(warm, T5B):
        eng.row_append(rows[t:t + 1])
    eng.flush()
    ph = np.zeros(10)
    nt3 = np.zeros(3, dtype=np.int64)
    lib.isvd_engine_phase_times(eng._h.h, ph.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                nt3.ctypes.data_as(i64p))
    lib.isvd_engine_set_timing(eng._h.h, 0)
    # end to end: pinned host rows, per-step D2H of the scalars
    h_rows = torch.empty((T5B, N5B), dtype=torch.float64, pin_memory=True)
    h_rows.copy_(rows)
    hr = h_rows.numpy()
    res = torch.empty((RES_SLOTS, 3), dtype=torch.float64, pin_memory=True)
    eng.restore()
    barrier()
    t0 = time.perf_counter()
    for t in range(warm, T5B):
        eng.row_append(hr[t:t + 1])
        # step result, read E2E_LAG steps behind its issue (as the 5a leg); every
        # result is read inside the timed region
        eng.scalars_async(res[t % RES_SLOTS].numpy(), t % RES_SLOTS)
        if t - warm >= E2E_LAG:
            eng.scalars_wait((t - E2E_LAG) % RES_SLOTS)
    for t in range(max(warm, T5B - E2E_LAG), T5B):
        eng.scalars_wait(t % RES_SLOTS)
    eng.flush()
    eng.synchronize()
    e2e_s = max_over_ranks(time.perf_counter() - t0, device=dev)
    window = int(lib.isvd_engine_lazy_window(eng._h.h))
    del eng
    torch.cuda.empty_cache()
    nrow = max(1, int(nt3[0]))
    per = {name: float(ph[j] / nrow) for j, name in enumerate(("project", "core_svd", "rotate",
                                                                "install"))}
    flush_ms, flush_bytes = float(ph[8]), float(ph[9])
    flush_flops = 2.0 * ml * K5B * K5B
    tick_ms = sum(per.values())
    summ, summ_file = _ncu_summary()
    traffic = summ.get("rot5b_flush", {}).get("dram_bytes") if world == 1 else None
    return {
        "metric": "iSVD updates/sec (k=128)", "value": steps / (ms / 1e3), "unit": UNIT,
        "steps": steps, "warmup": warm, "ms_per_step": ms / steps, "scaling": "strong",
        "config": {"workload": "cfg5b_tall", "m": M5B, "n": N5B, "rank": RANK5B, "k": K5B,
                   "row_appends": T5B, "noise_sd": 1e-3,
                   "parallelism": "1 GPU" if world == 1 else
                   f"U and A row-sharded over {world} GPUs (NCCL allreduce of Grams)",
                   "rows_per_gpu": ml, "deferred_u_rows": window},
        "gpu_launches": int(launches),
        "e2e": {"value": steps / e2e_s, "unit": UNIT, "h2d_bytes_per_step": N5B * 8,
                "d2h_bytes_per_step": 3 * 8, "steps": steps,
                "result_readback_lag_steps": E2E_LAG},
        "roofline": {"kernel": "rotate U flush (K3, deferred, DMMA)", "bound": "tensor",
                     "achieved": flush_flops / (flush_ms / 1e3) / 1e12 if flush_ms else None,
                     "peak": DMMA_PEAK_TFS, "unit": "TFLOP/s",
                     "frac": (flush_flops / (flush_ms / 1e3) / 1e12 / DMMA_PEAK_TFS)
                     if flush_ms else None,
                     "peak_kind": "measured FP64 DMMA (profiles/r01_fp64_peaks.txt)",
                     "traffic": traffic,
                     "traffic_source": f"profiles/{summ_file}: rot5b_flush (ncu)" if traffic
                     else None,
                     "hbm_gbs": flush_bytes / (flush_ms / 1e3) / 1e9 if flush_ms else None,
                     "flops_per_launch": flush_flops, "bytes_per_launch": flush_bytes},
        "phase_ms_per_tick": per,
        "flush_ms": flush_ms,
        "tick_busy_ms": tick_ms,
        "ortho_defect": [float(du), float(dv)],
        "init_s": init_s,
        "reference_hbm_ceiling_updates_per_s": 6553.3e9 / (8.0 * (2 * M5B * K5B + 2 * N5B * K5B
                                                                    + 2 * N5B)),
    }


def run_gpu(args):
    import ctypes

    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if os.environ.get("ISVD_BENCH_BACKEND", "nccl") != "nccl":
        local %= max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        # ISVD_BENCH_BACKEND=gloo: functional check of the N > 1 path with all
        # ranks on one GPU (not a measurement); NCCL otherwise
        backend = os.environ.get("ISVD_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    from paper_2605_24514_b200 import BatchedSvdEngine, _lib
    from paper_2605_24514_b200.sharding import max_over_ranks, shard_streams

    lib = _lib.load()
    i64p = ctypes.POINTER(ctypes.c_int64)
    total = args.streams
    streams = list(shard_streams(total, world, rank))
    B = len(streams)
    steps, warm = args.steps, args.warmup
    n_events = max(steps, warm)
    a0, rows, ii, jj, dd = make_inputs(torch, dev, streams, n_events=n_events)
    m_cap = M0 + (n_events + 1) // 2 + 1

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()

    res = torch.empty((RES_SLOTS, 3 * B), dtype=torch.float64, pin_memory=True)

    def run_ticks(eng, nt, host=None):
        """nt ticks; device-resident inputs unless host=(rows, ii, jj, dd).
        With host inputs every step's result (sq_norm, residual, input norm
        per stream) is read back to pinned host memory; the host waits for
        step t's result after issuing step t + E2E_LAG (the read-back lags by
        E2E_LAG steps; every result is read inside the timed region), so
        input validation and upload overlap the device's work."""
        for t in range(nt):
            if t % 2 == 0:
                eng.row_append(rows[t // 2] if host is None else host[0][t // 2])
            elif host is None:
                eng.rank_one_update(ii[t // 2], jj[t // 2], dd[t // 2])
            else:
                eng.rank_one_update(host[1][t // 2], host[2][t // 2], host[3][t // 2])
            if host is not None:
                eng.scalars_async(res[t % RES_SLOTS].numpy(), t % RES_SLOTS)
                if t >= E2E_LAG:
                    eng.scalars_wait((t - E2E_LAG) % RES_SLOTS)
        if host is not None and nt > 0:
            for t in range(max(0, nt - E2E_LAG), nt):
                eng.scalars_wait(t % RES_SLOTS)
            assert np.all(np.isfinite(res[(nt - 1) % RES_SLOTS].numpy()))

    t_init = time.perf_counter()
    eng = BatchedSvdEngine(a0, K, m_cap=m_cap, k_cap=K)
    if args.window:
        _lib.check(lib.isvd_engine_set_lazy_window(eng._h.h, args.window))
    eng.synchronize()
    init_s = time.perf_counter() - t_init
    eng.snapshot()
    # ---------------- warm-up (then back to the initial state)
    run_ticks(eng, warm)
    eng.flush()
    eng.restore()
    # ---------------- device-resident timing (value): grouped, no phase timing
    stream = torch.cuda.ExternalStream(eng.cuda_stream, device=dev)
    barrier()
    l0 = _lib.launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(str(ROOT / "gpurun_out" / f"clocks_r{rank}.csv")) as clk:
        torch.cuda.nvtx.range_push("isvd_timed")  # ncu --nvtx-include isvd_timed/
        e0.record(stream)
        run_ticks(eng, steps)
        eng.flush()  # materialise deferred U rotations inside the timed region
        e1.record(stream)
        torch.cuda.nvtx.range_pop()
        barrier()
    launches = _lib.launch_count() - l0
    dev_ms = e0.elapsed_time(e1)
    t_max = max_over_ranks(dev_ms, device=dev)
    value = total * steps / (t_max / 1e3)
    clock = clk.summary(local)
    f0 = eng.factors(0)
    assert np.all(np.isfinite(f0.s)) and np.all(np.diff(f0.s) <= 0)
    # ---------------- per-kernel breakdown (same ticks, one group, CUDA events
    # around every phase on the engine stream)
    diag_steps = min(steps, args.diag_steps)
    eng.restore()
    dbg = np.zeros(8, dtype=np.int64)
    _lib.check(lib.isvd_debug_counters(dbg.ctypes.data_as(i64p), 1))
    _lib.check(lib.isvd_engine_set_timing(eng._h.h, 1))
    d0, d1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    d0.record(stream)
    run_ticks(eng, diag_steps)
    eng.flush()
    d1.record(stream)
    torch.cuda.synchronize()
    diag_ms = d0.elapsed_time(d1)
    ph = np.zeros(10)
    nt3 = np.zeros(3, dtype=np.int64)
    _lib.check(lib.isvd_engine_phase_times(eng._h.h, _lib.dptr(ph), nt3.ctypes.data_as(i64p)))
    _lib.check(lib.isvd_engine_set_timing(eng._h.h, 0))
    _lib.check(lib.isvd_debug_counters(dbg.ctypes.data_as(i64p), 1))
    n_flush = int(nt3[2])
    flush_ms, flush_bytes = float(ph[8]), float(ph[9])
    phase_by_kind = {
        kind: {name: float(ph[4 * i + j] / max(1, nt3[i]))
               for j, name in enumerate(("project", "core_svd", "rotate", "install"))}
        for i, kind in enumerate(("row_append", "rank_one"))}
    window = int(lib.isvd_engine_lazy_window(eng._h.h))
    proj_bytes, rot_row, rot_r1, vflush_bytes, _ = _simulate_bytes(B, diag_steps, window)
    all_bytes = _simulate_bytes(B, steps, window)[4]
    # ---------------- end-to-end through the public API with host buffers
    e2e_steps = min(steps, args.e2e_steps)
    nrow = (e2e_steps + 1) // 2
    nr1 = e2e_steps // 2
    h_rows = torch.empty((nrow, B, N0), dtype=torch.float64, pin_memory=True)
    h_rows.copy_(rows[:nrow])
    h_ii = torch.empty((nr1, B), dtype=torch.int64, pin_memory=True)
    h_jj = torch.empty((nr1, B), dtype=torch.int64, pin_memory=True)
    h_dd = torch.empty((nr1, B), dtype=torch.float64, pin_memory=True)
    h_ii.copy_(ii[:nr1]); h_jj.copy_(jj[:nr1]); h_dd.copy_(dd[:nr1])
    host = (h_rows.numpy(), h_ii.numpy(), h_jj.numpy(), h_dd.numpy())
    eng.restore()
    barrier()
    t0 = time.perf_counter()
    run_ticks(eng, e2e_steps, host=host)
    eng.flush()
    barrier()
    e2e_s = max_over_ranks(time.perf_counter() - t0, device=dev)
    e2e_value = total * e2e_steps / e2e_s
    h2d = (nrow * B * N0 * 8 + nr1 * B * 24) / max(1, e2e_steps)
    d2h = 3 * B * 8
    del eng
    del a0, rows, ii, jj, dd
    torch.cuda.empty_cache()
    k128 = None
    if not args.no_k128:
        k128 = run_cfg5b(torch, dev, lib, warm, world, rank)

    if rank == 0:
        peak, peak_kind = _peaks()
        tot = lambda i: float(ph[i] + ph[4 + i])
        # the deferred-basis rotations run inside the core kernels (warp DMMA
        # epilogues), so their bytes are accounted with them
        kernels = {
            "project_append (K1, row ticks)": {"ms": float(ph[0]), "bytes": proj_bytes},
            "append core + fused W/G rotation (K2a, row ticks)": {
                "ms": float(ph[1] + ph[2]), "bytes": rot_row},
            "rank-1 core + fused W/G rotation (K2b, rank-1 ticks)": {
                "ms": float(ph[4] + ph[5] + ph[6]), "bytes": rot_r1},
            "rotate U flush (K3, deferred)": {"ms": flush_ms, "bytes": flush_bytes},
            "V materialisation (K3, every 8 row appends)": {"ms": max(0.0, tot(3) - flush_ms),
                                                            "bytes": vflush_bytes or None},
        }
        busy = sum(v["ms"] for v in kernels.values())
        for v in kernels.values():
            v["share"] = v["ms"] / busy if busy else None
            v["ms_per_step"] = v["ms"] / max(1, diag_steps)
            v["gbs"] = (v["bytes"] / (v["ms"] / 1e3) / 1e9) if (v["bytes"] and v["ms"]) else None
        # algorithmic flops of the two FP64-latency-bound core kernels
        r1_steps = float(dbg[6]) / max(1, int(dbg[7])) if dbg[7] else 2.0
        f_r1, f_row = _simulate_flops(B, diag_steps, window, rank1_steps=r1_steps)
        kernels["rank-1 core + fused W/G rotation (K2b, rank-1 ticks)"]["flops"] = f_r1
        kernels["append core + fused W/G rotation (K2a, row ticks)"]["flops"] = f_row
        for v in kernels.values():
            v["tflops"] = (v["flops"] / (v["ms"] / 1e3) / 1e12) if (v.get("flops") and v["ms"]) \
                else None
        flush_k = kernels["rotate U flush (K3, deferred)"]
        flush_k["flops"] = 2.0 * B * M0 * K * K * n_flush if n_flush else None
        summ, summ_file = _ncu_summary()

        def ncu_traffic(key):
            # captures are one stream-group launch (B / 4 streams); scaled to all B
            if key in summ and "dram_bytes" in summ[key]:
                return summ[key]["dram_bytes"] * 4.0 * B / TOTAL_STREAMS
            return None

        # roofline of the dominant kernel by time, against the resource that
        # binds it: K1 and the rotations stream HBM; the core kernels run on
        # the FP64 pipes (DMMA for the Gram / rotation products, DFMA for the
        # secular solve), so their roof is the measured DMMA peak
        dom_name = max(kernels, key=lambda k: kernels[k]["ms"])
        dom = kernels[dom_name]
        n_launch = max(1, (diag_steps + 1) // 2 if "row ticks" in dom_name else diag_steps // 2)
        ncu_key = {"project_append (K1, row ticks)": "proj5a",
                   "append core + fused W/G rotation (K2a, row ticks)": "arrowcta",
                   "rank-1 core + fused W/G rotation (K2b, rank-1 ticks)": "r1fast"}.get(dom_name)
        traffic = ncu_traffic(ncu_key) if ncu_key else None
        measured = (f"first {diag_steps} ticks in timing mode (one launch per kernel over all "
                    "streams, CUDA events around each phase on the engine stream)")
        if dom.get("flops"):
            roof = {"kernel": dom_name, "bound": "tensor", "achieved": dom["tflops"],
                    "peak": DMMA_PEAK_TFS, "unit": "TFLOP/s", "frac": dom["tflops"] / DMMA_PEAK_TFS,
                    "peak_kind": "measured FP64 DMMA.8x8x4 peak (profiles/r01_fp64_peaks.txt); "
                                 "FP64 has no tcgen05 kind",
                    "flops_per_launch": dom["flops"] / n_launch,
                    "bytes_per_launch": dom["bytes"] / n_launch,
                    "hbm_frac": dom["gbs"] / peak if dom.get("gbs") else None}
        else:
            roof = {"kernel": dom_name, "bound": "hbm", "achieved": dom["gbs"], "peak": peak,
                    "unit": "GB/s", "frac": dom["gbs"] / peak, "peak_kind": peak_kind,
                    "bytes_per_launch": dom["bytes"] / n_launch}
        roof.update({"traffic": traffic,
                     "traffic_source": f"profiles/{summ_file}: {ncu_key} dram__bytes_read+write of "
                                       "one stream-group launch x 4 groups (ncu, cold cache)"
                     if traffic else None,
                     "launch": "one launch over all streams of the GPU",
                     "measured_over": measured})
        if ncu_key and ncu_key in summ:
            roof["ncu"] = {k2: summ[ncu_key].get(k2) for k2 in
                           ("fp64_pipe_pct", "dmma_pipe_pct", "occupancy_pct", "dram_pct_peak",
                            "regs", "warp_instructions", "tensor_fp64_ops")}
            # executed (not algorithmic) FP64 tensor work: ncu's
            # sm__ops_path_tensor_src_fp64.sum of one stream-group launch,
            # scaled to all streams, over this run's measured launch time --
            # the share of the DMMA roof the kernel actually occupies (symmetric
            # products computed in full tiles, 8-row group padding and the
            # convergence-check Grams are executed but not algorithmic flops)
            t_ops = summ[ncu_key].get("tensor_fp64_ops")
            if t_ops and dom["ms"]:
                ex = t_ops * 4.0 * B / TOTAL_STREAMS * n_launch / (dom["ms"] / 1e3) / 1e12
                roof["executed"] = {"tensor_tflops": ex, "frac_of_dmma_peak": ex / DMMA_PEAK_TFS,
                                    "source": f"profiles/{summ_file}: {ncu_key} "
                                              "sm__ops_path_tensor_src_fp64.sum x 4 groups"}
        # BASELINE's second metric: basis-rotation HBM GB/s -- the deferred U
        # flush and the V materialisation, the two launches that stream a
        # tall basis through HBM
        rot_k = kernels["rotate U flush (K3, deferred)"]
        vm_k = kernels["V materialisation (K3, every 8 row appends)"]
        rotation = {
            "metric": "basis-rotation HBM GB/s", "unit": "GB/s", "peak": peak,
            "u_flush": {"achieved": rot_k["gbs"], "frac": rot_k["gbs"] / peak if rot_k["gbs"] else None,
                        "bytes": rot_k["bytes"], "ms": rot_k["ms"], "launches": n_flush,
                        "traffic": ncu_traffic("flush5a")},
            "v_materialisation": {"achieved": vm_k["gbs"],
                                  "frac": vm_k["gbs"] / peak if vm_k["gbs"] else None,
                                  "bytes": vm_k["bytes"], "ms": vm_k["ms"],
                                  "traffic": ncu_traffic("vflush5a")},
            "k1_projection": {"achieved": kernels["project_append (K1, row ticks)"]["gbs"],
                              "frac": kernels["project_append (K1, row ticks)"]["gbs"] / peak},
        }
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": steps,
            "warmup": warm, "ms_per_step": t_max / steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "cfg5a_batched_streams", "streams": total,
                       "streams_per_gpu": B, "m0": M0, "n": N0, "rank": RANK, "k": K,
                       "events": steps, "event_mix": "alternating row append / rank-1",
                       "l2": "inputs larger than L2 (state ~2 GB/GPU touched per step)",
                       "parallelism": f"streams sharded over {world} GPU(s)",
                       "deferred_u_rows": window, "stream_groups": 4},
            "clocks": clock,
            "gpu_launches": int(launches),
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h), "steps": e2e_steps,
                    "result_readback_lag_steps": E2E_LAG},
            "roofline": roof,
            "rotation": rotation,
            "kernels": kernels,
            "flushes": n_flush,
            "phase_ms_by_event": phase_by_kind,
            # the reference algorithm's compulsory bytes per second of
            # this run: a throughput in the reference's units, NOT an achieved
            # bandwidth (the deferred bases move far fewer bytes)
            "reference_algorithm_bytes_rate_gbs": all_bytes / (t_max / 1e3) / 1e9,
            "diagnostics": {"jacobi32_sweeps_per_core": float(dbg[0]) / max(1, int(dbg[1])),
                            "rank1_fast_path_fraction": float(dbg[7]) / max(1, int(dbg[1])),
                            "rank1_steps_per_core": float(dbg[6]) / max(1, int(dbg[1])),
                            "init_s": init_s,
                            "serial_phase_ms_per_step": diag_ms / max(1, diag_steps)},
        }
        if k128 is not None:
            line["k128"] = k128
        if world == 1 and not args.no_cpu_baseline:
            v, cores, updates, secs = cpu_reference(args.cpu_streams, args.cpu_events)
            line["cpu_baseline"] = {
                "value": v, "unit": UNIT, "cores": cores, "kind": "port",
                "sample": f"{args.cpu_streams} cfg5a streams x {args.cpu_events} events on "
                          f"{cores} processes (oracle/ numpy restatement, 1 BLAS thread each, "
                          f"init excluded)"}
            if k128 is not None:
                v5, c5, t5, s5 = cpu_reference_5b()
                k128["cpu_baseline"] = {
                    "value": v5, "unit": UNIT, "cores": c5, "kind": "port",
                    "sample": f"{t5} full-size row appends through the oracle row-append "
                              "kernel (numpy/BLAS, all host threads), engine vstack excluded"}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=EVENTS)
    ap.add_argument("--warmup", type=int, default=8)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--streams", type=int, default=TOTAL_STREAMS)
    ap.add_argument("--e2e-steps", type=int, default=512)
    ap.add_argument("--diag-steps", type=int, default=256)
    ap.add_argument("--cpu-streams", type=int, default=64)
    ap.add_argument("--cpu-events", type=int, default=EVENTS)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-k128", action="store_true", help="skip the config-5b (k=128) leg")
    ap.add_argument("--window", type=int, default=0,
                    help="deferred-U window for config 5a (0 = the engine default)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    (ROOT / "gpurun_out").mkdir(exist_ok=True)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()

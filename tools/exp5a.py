"""Config-5a tick-rate experiments (not a test): ms per tick for engine knobs.

  python tools/exp5a.py [--streams 4096] [--ticks 256] [--groups 1,4,8]
Each configuration restores the same snapshot and times `ticks` device-
resident ticks (alternating row append / rank-1) with CUDA events."""
import argparse
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2605_24514_b200 import BatchedSvdEngine, _lib  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--streams", type=int, default=4096)
    ap.add_argument("--ticks", type=int, default=256)
    ap.add_argument("--groups", default="4")
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--e2e", action="store_true", help="also time the pinned-host loop")
    ap.add_argument("--lags", default="1", help="result read-back lag(s) of the host loop")
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    lib = _lib.load()
    a0, rows, ii, jj, dd = bench.make_inputs(torch, dev, list(range(args.streams)),
                                             n_events=args.ticks)
    eng = BatchedSvdEngine(a0, bench.K, m_cap=bench.M0 + args.ticks // 2 + 2, k_cap=bench.K)
    del a0
    eng.synchronize()
    eng.snapshot()
    stream = torch.cuda.ExternalStream(eng.cuda_stream, device=dev)

    def run(nt):
        for t in range(nt):
            if t % 2 == 0:
                eng.row_append(rows[t // 2])
            else:
                eng.rank_one_update(ii[t // 2], jj[t // 2], dd[t // 2])
        eng.flush()

    def pinned(x):
        h = torch.empty(x.shape, dtype=x.dtype, pin_memory=True)
        h.copy_(x)
        return h.numpy()

    if args.e2e:
        import time
        hr, hi, hj, hd = (pinned(x) for x in (rows, ii, jj, dd))
        res = torch.empty((8, 3 * args.streams), dtype=torch.float64, pin_memory=True)

        def run_host(nt, lag):
            for t in range(nt):
                if t % 2 == 0:
                    eng.row_append(hr[t // 2])
                else:
                    eng.rank_one_update(hi[t // 2], hj[t // 2], hd[t // 2])
                eng.scalars_async(res[t % 8].numpy(), t % 8)
                if t >= lag:
                    eng.scalars_wait((t - lag) % 8)
            for t in range(max(0, nt - lag), nt):
                eng.scalars_wait(t % 8)
            eng.flush()
            eng.synchronize()

    for g in [int(x) for x in args.groups.split(",")]:
        _lib.check(lib.isvd_engine_set_groups(eng._h.h, g))
        best = None
        for _ in range(args.reps):
            eng.restore()
            run(16)
            eng.restore()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            run(args.ticks)
            e1.record(stream)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / args.ticks
            best = ms if best is None else min(best, ms)
        msg = f"groups={g}: {best:.4f} ms/tick  {args.streams / best / 1e3:.3f} M updates/s"
        for lag in ([int(x) for x in args.lags.split(",")] if args.e2e else []):
            eng.restore()
            run_host(16, lag)
            eng.restore()
            eng.synchronize()
            t0 = time.perf_counter()
            run_host(args.ticks, lag)
            ms = (time.perf_counter() - t0) * 1e3 / args.ticks
            msg += f" | e2e lag {lag}: {ms:.4f} ms/tick {args.streams / ms / 1e3:.3f} M/s"
        print(msg, flush=True)


if __name__ == "__main__":
    main()

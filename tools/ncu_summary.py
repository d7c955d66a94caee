"""Summarise ncu artefacts into profiles/ (run here, after gpurun).

  python tools/ncu_summary.py <tag>
reads gpurun_out/launches.csv and gpurun_out/*.ncu-rep, writes
profiles/<tag>_launches.txt (per-kernel share of the bench launch list) and
profiles/<tag>_ncu_summary.json (duration, DRAM bytes, throughputs, pipe
utilisation per captured kernel)."""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
OUT = ROOT / "gpurun_out"
tag = sys.argv[1] if len(sys.argv) > 1 else "r01"

KEYS = {
    "gpu__time_duration.sum": "duration_ns",
    "dram__bytes_read.sum": "dram_read_bytes",
    "dram__bytes_write.sum": "dram_write_bytes",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct_peak",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed": "mem_pct_peak",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct_peak",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active": "fp64_pipe_pct",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_cycles_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occupancy_pct",
    "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active": "dmma_pipe_pct",
    "sm__ops_path_tensor_src_fp64.avg.pct_of_peak_sustained_elapsed": "tensor_fp64_ops_pct_peak",
    "sm__ops_path_tensor_src_fp64.sum": "tensor_fp64_ops",
    "TPC.TriageCompute.sm__pipe_fp64_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed": "fp64_cycles_realtime_pct",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio": "stall_wait_per_issue",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "launch__registers_per_thread": "regs",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "smsp__inst_executed.sum": "warp_instructions",
    "lts__t_bytes.sum": "l2_bytes",
}


def launches():
    p = OUT / "launches.csv"
    if not p.exists():
        return None
    rows = [r for r in csv.reader(io.StringIO(p.read_text())) if len(r) > 10]
    h = rows[0]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        name = r[ki].split("(")[0].replace("void ", "").split("::")[-1]
        agg[name][0] += 1
        agg[name][1] += float(r[vi].replace(",", ""))
    tot = sum(v[1] for v in agg.values())
    lines = [f"ncu launch list (gpu__time_duration.sum, --clock-control none; cold-cache, "
             f"serialised), NVTX range isvd_timed of: python bench.py --steps 16 --warmup 3 "
             f"--no-k128 (the device-resident timed ticks only)",
             f"{'kernel':40s} {'launches':>8s} {'total us':>10s} {'share':>6s}"]
    for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"{k:40s} {c:8d} {t / 1e3:10.1f} {t / tot:6.3f}")
    return "\n".join(lines) + "\n"


def rep(path):
    res = subprocess.run(["ncu", "-i", str(path), "--page", "raw", "--csv"], capture_output=True,
                         text=True)
    rows = list(csv.reader(io.StringIO(res.stdout)))
    if len(rows) < 3:
        return None
    h, units, row = rows[0], rows[1], rows[2]
    out = {"kernel": row[h.index("Kernel Name")][:120] if "Kernel Name" in h else None}
    scale = {"nsecond": 1.0, "usecond": 1e3, "msecond": 1e6, "second": 1e9,
             "ns": 1.0, "us": 1e3, "ms": 1e6, "s": 1e9,
             "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    for k, name in KEYS.items():
        if k in h:
            i = h.index(k)
            v = row[i].replace(",", "")
            try:
                out[name] = float(v) * scale.get(units[i], 1.0)
            except ValueError:
                out[name] = v
    if "dram_read_bytes" in out and "dram_write_bytes" in out:
        out["dram_bytes"] = out["dram_read_bytes"] + out["dram_write_bytes"]
        if out.get("duration_ns"):
            out["dram_gbs"] = out["dram_bytes"] / out["duration_ns"]  # bytes/ns = GB/s
    return out


def main():
    import os
    prof = Path(os.environ.get("ISVD_SUMMARY_OUT", str(ROOT / "profiles")))
    txt = launches()
    if txt:
        (prof / f"{tag}_launches.txt").write_text(txt)
        print(txt)
    summ = {}
    for p in sorted(OUT.glob("*.ncu-rep")):
        r = rep(p)
        if r:
            summ[p.stem] = r
    (prof / f"{tag}_ncu_summary.json").write_text(json.dumps(summ, indent=1))
    print(json.dumps(summ, indent=1))


if __name__ == "__main__":
    main()

"""Per-source-line warp-stall samples and executed instructions of one
kernel in an ncu report, by mapping SASS offsets to -lineinfo lines of a
locally compiled cubin (same flags as the library):
  python tools/ncu_lines.py gpurun_out/x.ncu-rep csrc/file.cu kernel_substring [top]"""
import csv
import io
import re
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
rep, src, kname = sys.argv[1], sys.argv[2], sys.argv[3]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
cubin = "/tmp/ncu_lines.cubin"
subprocess.run(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3",
                "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
                f"-I{ROOT / 'include'}", f"-I{ROOT / 'paper_2605_24514_b200/csrc'}", "-cubin", "-o",
                cubin, str(ROOT / "paper_2605_24514_b200/csrc" / src)]
               + (["-rdc=true"] if src in ("core_svd.cu", "arrow_svd.cu") else []), check=True)
sass = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
lines = sass.split("\n")
start = next(i for i, l in enumerate(lines) if l.strip().startswith(".text.") and kname in l)
addr2line, cur = {}, None
for l in lines[start + 1:]:
    if l.strip().startswith(".text."):
        break
    m = re.search(r'//## File "(.*)", line (\d+)', l)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*)", l)
    if m:
        addr2line[int(m.group(1), 16)] = cur
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, data = rows[1], rows[2:]
base = int(data[0][0], 16)
si, ie = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
agg, ts, ti = {}, 0, 0
for r in data:
    ln = addr2line.get(int(r[0], 16) - base)
    s, n = int(r[si] or 0), int(float(r[ie] or 0))
    ts, ti = ts + s, ti + n
    a = agg.setdefault(ln, [0, 0])
    a[0] += s
    a[1] += n
print(f"samples {ts}, warp instructions {ti}")
srcs = {}
for k, v in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
    txt = ""
    if k:
        p = ROOT / "paper_2605_24514_b200/csrc" / k[0]
        if p.exists():
            srcs.setdefault(k[0], p.read_text().split("\n"))
            txt = srcs[k[0]][k[1] - 1].strip()[:70]
    print(f"{str(k):32s} {v[0]:5d} {100 * v[0] / ts:5.1f}% {v[1]:9d}  {txt}")

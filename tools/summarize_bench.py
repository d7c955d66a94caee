"""Print the key fields of a bench.py JSON line (file or stdin)."""
import json
import signal
import sys

signal.signal(signal.SIGPIPE, signal.SIG_DFL)

src = open(sys.argv[1]).read() if len(sys.argv) > 1 else sys.stdin.read()
line = [l for l in src.splitlines() if l.startswith('{"metric"') or l.startswith('{"impl"')][-1]
d = json.loads(line)
print("value", round(d["value"]), "ms/step", round(d["ms_per_step"], 4), "e2e", round(d.get("e2e", {}).get("value", 0)))
for k, v in d.get("kernels", {}).items():
    print(f"  {k:45s} {v['ms_per_step']:.4f} ms/step  share {v['share']:.3f}  gbs {v['gbs'] and round(v['gbs'])}")
print("  by event:", json.dumps(d.get("phase_ms_by_event")))
print("  roofline:", json.dumps(d.get("roofline")))
if "diagnostics" in d:
    print("  diagnostics:", json.dumps(d["diagnostics"]))

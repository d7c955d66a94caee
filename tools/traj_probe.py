"""Run a stored reference stream (tests/golden) through the product loop on
the GPU and save the trajectory + per-tick orthonormality defects for
offline comparison: python tools/traj_probe.py cfg1 cfg2"""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
from conftest import sim_array, sim_inputs  # noqa: E402
from paper_2605_24514_b200 import workloads  # noqa: E402
from paper_2605_24514_b200.policies import AdaptiveRankConfig, PolicyConfig  # noqa: E402
from paper_2605_24514_b200.stream import run_stream  # noqa: E402

golden = np.load(ROOT / "tests/golden/reference_golden.npz")
out = {}
for tag in sys.argv[1:]:
    a0, ev, k, pol, log_every = sim_inputs(golden, tag)
    ad = pol.pop("adaptive", None)
    policy = PolicyConfig(**pol, adaptive=AdaptiveRankConfig(**ad) if ad else None)
    recs, eng = run_stream(a0, workloads.to_stream_events(ev), k, policy, log_every,
                           return_engine=True)
    out[f"{tag}_records"] = sim_array(recs)
    out[f"{tag}_u"] = eng.factors.u
    out[f"{tag}_defects"] = np.array(eng.ortho_defects())
    print(tag, "defects", eng.ortho_defects(), flush=True)
(ROOT / "gpurun_out").mkdir(exist_ok=True)
np.savez(ROOT / "gpurun_out" / "traj_probe.npz", **out)

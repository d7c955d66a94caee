"""GPU oracle basis and principal-angle accuracy on config 2's matrix after
some rank-1 events (vs LAPACK): python tools/angle_probe.py"""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from oracle import OracleEngine, principal_angle_max  # noqa: E402
from paper_2605_24514_b200 import SvdEngine, workloads  # noqa: E402
from paper_2605_24514_b200.metrics import angle_to_opt, compute_oracle  # noqa: E402

a0, ev, _ = workloads.cfg2(0, n_events=266)
g, c = SvdEngine(a0, 20), OracleEngine(a0, 20)
for e in ev:
    g.rank_one_update(*e[1:])
    c.rank_one_update(*e[1:])
A = c.tracked
og = compute_oracle(g, 20)
U, S, Vt = np.linalg.svd(A, full_matrices=False)
Ub = U[:, :20]
def sine(q1, q2):
    r = q2 - q1 @ (q1.T @ q2)
    return np.linalg.norm(r, 2)
print("gpu oracle basis vs lapack: sine", sine(og.basis, Ub), "defect",
      np.linalg.norm(og.basis.T @ og.basis - np.eye(20)))
print("sigma rel", np.max(np.abs(og.singular_values - S) / S))
fu = g.factors.u
print("gpu U vs cpu U sine", sine(fu, c.factors.u))
print("angle gpu (gpu basis)", angle_to_opt(g, og.basis))
print("angle gpu (lapack basis)", angle_to_opt(g, Ub))
print("angle numpy(gpu U, lapack basis)", principal_angle_max(fu, Ub))
print("angle numpy(cpu U, lapack basis)", principal_angle_max(c.factors.u, Ub))
print("angle numpy(gpu U, gpu basis)", principal_angle_max(fu, og.basis))

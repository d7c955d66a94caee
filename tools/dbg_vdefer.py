import sys; sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import numpy as np
from paper_2605_24514_b200 import SvdEngine, frob_error
from test_gpu_vdefer import _mixed_events, _apply
k = int(sys.argv[1]) if len(sys.argv) > 1 else 5
rng = np.random.default_rng(100 + k)
m0, n0 = 90, 50
a0 = rng.standard_normal((m0, n0)) @ np.diag(np.logspace(0, -2, n0)) @ rng.standard_normal((n0, n0))
events = _mixed_events(rng, 160, m0, n0)
for T in range(1, 40):
    dfr, eag = SvdEngine(a0, k), SvdEngine(a0, k)
    dfr.set_vdefer(2); eag.set_vdefer(0)
    for t in range(T):
        _apply(dfr, events[t]); _apply(eag, events[t])
    d = abs(frob_error(dfr) - frob_error(eag)) / frob_error(eag)
    s = np.max(np.abs(dfr.factors.s - eag.factors.s) / eag.factors.s)
    print(T, events[T-1][0], f"{d:.2e} {s:.2e}", dfr.factors.rank)
    if d > 1e-9: break

"""Seeded synthetic inputs for the BASELINE.json configurations.

BASELINE.json defines its own synthetic workloads; these
generators write them.  Seeds fan out into numpy PCG64 substreams
``default_rng([seed, config, lane])`` (the pattern of svdstream/rng.py:11-24)
so extending a stream never perturbs earlier draws.

Events are tuples: ("row", x) | ("col", y) | ("rank1", i, j, delta).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


def _rng(seed: int, cfg: int, lane: int) -> np.random.Generator:
    return np.random.default_rng([int(seed), int(cfg), int(lane)])


def cfg1(seed: int = 0, n_events: int = 1000):
    """Row-append stream: A0 = U0 V0^T + N(0, 0.1^2) (200 x 100, rank 10);
    rows x = u V0^T + N(0, 0.1^2 I); k = 10, periodic refresh every 100,
    metrics every tick."""
    g = _rng(seed, 1, 0)
    u0 = g.standard_normal((200, 10))
    v0 = g.standard_normal((100, 10))
    a0 = u0 @ v0.T + 0.1 * g.standard_normal((200, 100))
    ge = _rng(seed, 1, 1)
    events = []
    for _ in range(n_events):
        u = ge.standard_normal(10)
        events.append(("row", v0 @ u + 0.1 * ge.standard_normal(100)))
    return a0, events, dict(k=10, policy=dict(kind="periodic", period=100), log_every=1)


def cfg2(seed: int = 0, n_events: int = 10_000):
    """Rank-1 stream: A0 = X Y^T + N(0, 0.1^2) (1000 x 500, rank 20);
    (i, j) uniform, delta ~ N(0, (0.1 rms(A0))^2); k = 20, error refresh at 1.05."""
    g = _rng(seed, 2, 0)
    x = g.standard_normal((1000, 20))
    y = g.standard_normal((500, 20))
    a0 = x @ y.T + 0.1 * g.standard_normal((1000, 500))
    rms = float(np.sqrt(np.mean(a0 * a0)))
    ge = _rng(seed, 2, 1)
    ii = ge.integers(0, 1000, size=n_events)
    jj = ge.integers(0, 500, size=n_events)
    dd = ge.normal(0.0, 0.1 * rms, size=n_events)
    events = [("rank1", int(i), int(j), float(d)) for i, j, d in zip(ii, jj, dd)]
    return a0, events, dict(k=20, policy=dict(kind="error", gamma=1.05, min_spacing=0),
                            log_every=1)


def cfg3(seed: int = 0, t_total: int = 2520, n_assets: int = 50, t0: int = 252):
    """Synthetic 5-factor return panel, full-sample mean-centred; init on
    the first 252 rows then one row append per day; k = 5, angle refresh 5 deg."""
    g = _rng(seed, 3, 0)
    f = g.normal(0.0, 0.01, size=(t_total, 5))
    load = np.empty((n_assets, 5))
    load[:, 0] = g.normal(1.0, 0.3, size=n_assets)
    load[:, 1:] = g.normal(0.0, 0.5, size=(n_assets, 4))
    eps = 0.005 * g.standard_t(4, size=(t_total, n_assets))
    r = f @ load.T + eps
    r = r - r.mean(axis=0, keepdims=True)
    events = [("row", r[t].copy()) for t in range(t0, t_total)]
    return r[:t0].copy(), events, dict(k=5, policy=dict(kind="angle", theta_max=float(np.deg2rad(5.0))),
                                       log_every=1, panel=r)


def cfg4(seed: int = 0, m: int = 20_000, n: int = 5_000, rank: int = 64, n_blocks: int = 1000):
    """Large mixed stream: A0 = X diag(0.9^i) Y^T + N(0, 0.01^2); then
    n_blocks x (5 row appends, 1 column append) from the same factor model
    (coherent left/right loadings as svdstream/stream.py:151-164)."""
    g = _rng(seed, 4, 0)
    sig = 0.9 ** np.arange(rank)
    x = g.standard_normal((m, rank))
    y = g.standard_normal((n, rank))
    a0 = (x * sig) @ y.T + 0.01 * g.standard_normal((m, n))
    ge = _rng(seed, 4, 1)
    events = []
    rows = [x]
    cols = [y]
    xcur, ycur = x, y
    for _ in range(n_blocks):
        for _ in range(5):
            l = ge.standard_normal(rank)
            events.append(("row", ycur @ (sig * l) + 0.01 * ge.standard_normal(ycur.shape[0])))
            xcur = np.vstack([xcur, l[None, :]])
        l = ge.standard_normal(rank)
        events.append(("col", xcur @ (sig * l) + 0.01 * ge.standard_normal(xcur.shape[0])))
        ycur = np.vstack([ycur, l[None, :]])
    return a0, events, dict(k=64, policy=dict(kind="periodic", period=500,
                                              adaptive=dict(tau=0.95, k_min=1, k_max=128, eta=0.5)),
                            log_every=250)


def cfg5a_stream(seed: int, b: int, m: int = 1024, n: int = 256, rank: int = 32,
                 n_events: int = 1024):
    """One stream of the batched workload: A0 = X_b Y_b^T + N(0, 0.05^2),
    events alternating row append (l Y_b^T + N(0, 0.05^2)) and rank-1
    (i uniform over the current rows, j uniform, delta ~ N(0, 0.01))."""
    g = _rng(seed, 5, b)
    x = g.standard_normal((m, rank))
    y = g.standard_normal((n, rank))
    a0 = x @ y.T + 0.05 * g.standard_normal((m, n))
    events = []
    rows = m
    for t in range(n_events):
        if t % 2 == 0:
            l = g.standard_normal(rank)
            events.append(("row", y @ l + 0.05 * g.standard_normal(n)))
            rows += 1
        else:
            events.append(("rank1", int(g.integers(0, rows)), int(g.integers(0, n)),
                           float(g.normal(0.0, 0.01))))
    return a0, events


def cfg5a_batch(seed: int, batch: int, m: int = 1024, n: int = 256, rank: int = 32,
                n_events: int = 1024):
    """Host-side batch for parity tests: A0 (B, m, n) and per-tick event
    arrays (rows: (B, n) per even tick; rank-1: (I, J, D) per odd tick)."""
    streams = [cfg5a_stream(seed, b, m, n, rank, n_events) for b in range(batch)]
    a0 = np.stack([s[0] for s in streams])
    ticks = []
    for t in range(n_events):
        if t % 2 == 0:
            ticks.append(("row", np.stack([s[1][t][1] for s in streams])))
        else:
            ticks.append(("rank1", np.array([s[1][t][1] for s in streams], dtype=np.int64),
                          np.array([s[1][t][2] for s in streams], dtype=np.int64),
                          np.array([s[1][t][3] for s in streams])))
    return a0, ticks, streams


def to_stream_events(events):
    """Convert tuple events into stream.RowAppend / ColAppend / RankOneUpdate."""
    from .stream import ColAppend, RankOneUpdate, RowAppend

    out = []
    for ev in events:
        if ev[0] == "row":
            out.append(RowAppend(ev[1]))
        elif ev[0] == "col":
            out.append(ColAppend(ev[1]))
        else:
            out.append(RankOneUpdate(ev[1], ev[2], ev[3]))
    return out


# ---------------------------------------------------------------------------
# The reference's own synthetic streams (svdstream/stream.py:73-200 and
# rng.py), restated so its CLI scenarios and acceptance streams (which are
# calibrated on STREAM_SEED = 7, acceptance.py:35-37) can be replayed on the
# device engine.  Substream tags as rng.py:12-17.
INIT, EVENTS, STRUCTURAL, MIXED, PANEL, PORTFOLIO = 0, 1, 2, 3, 4, 5


def substream(seed: int, tag: int) -> np.random.Generator:
    """rng.py:20-25."""
    seed = int(seed)
    if seed < 0:
        raise ValueError(f"seed must be nonnegative, got {seed}")
    return np.random.default_rng([seed, int(tag)])


def gen_low_rank(m: int, n: int, rank: int, noise_scale: float, seed: int) -> np.ndarray:
    """stream.py:73-83: Gaussian factors of the given rank plus dense noise."""
    if not 1 <= rank <= min(m, n):
        raise ValueError(f"rank must be in [1, min(m, n)], got {rank} for {m}x{n}")
    if noise_scale < 0.0:
        raise ValueError(f"noise_scale must be >= 0, got {noise_scale}")
    gen = substream(seed, INIT)
    left = gen.standard_normal((m, rank))
    right = gen.standard_normal((n, rank))
    return left @ right.T + noise_scale * gen.standard_normal((m, n))


def gen_rank_one_events(count: int, delta_sd: float, rows: int, cols: int, seed: int):
    """stream.py:86-100: uniform in-bounds (i, j), normal deltas."""
    if count < 0:
        raise ValueError(f"count must be >= 0, got {count}")
    gen = substream(seed, EVENTS)
    i_idx = gen.integers(0, rows, size=count)
    j_idx = gen.integers(0, cols, size=count)
    deltas = gen.normal(0.0, delta_sd, size=count)
    return [("rank1", int(i), int(j), float(d)) for i, j, d in zip(i_idx, j_idx, deltas)]


def gen_structural_events(kind: str, count: int, factor_rank: int, noise_scale: float,
                          width: int, seed: int):
    """stream.py:103-127: appends from a fixed latent factor model."""
    if kind not in ("row", "col"):
        raise ValueError(f"kind must be 'row' or 'col', got {kind!r}")
    if count < 0:
        raise ValueError(f"count must be >= 0, got {count}")
    gen = substream(seed, STRUCTURAL)
    directions = gen.standard_normal((factor_rank, width))
    events = []
    for _ in range(count):
        loading = gen.standard_normal(factor_rank)
        events.append((kind, loading @ directions + noise_scale * gen.standard_normal(width)))
    return events


def gen_mixed_stream(count: int, mix_weights, base_m: int, base_n: int, factor_rank: int,
                     noise_scale: float, delta_sd: float, seed: int):
    """stream.py:130-165: weighted interleaving with coherent loadings."""
    weights = np.asarray(mix_weights, dtype=np.float64)
    if weights.shape != (3,) or np.any(weights < 0) or weights.sum() <= 0:
        raise ValueError("mix_weights must be 3 nonnegative values, not all zero")
    gen = substream(seed, MIXED)
    kinds = gen.choice(3, size=count, p=weights / weights.sum())
    left = gen.standard_normal((base_m, factor_rank))
    right = gen.standard_normal((base_n, factor_rank))
    events = []
    for kind in kinds:
        if kind == 0:
            loading = gen.standard_normal(factor_rank)
            events.append(("row", loading @ right.T + noise_scale * gen.standard_normal(len(right))))
            left = np.vstack([left, loading[None, :]])
        elif kind == 1:
            loading = gen.standard_normal(factor_rank)
            events.append(("col", left @ loading + noise_scale * gen.standard_normal(len(left))))
            right = np.vstack([right, loading[None, :]])
        else:
            i = int(gen.integers(0, len(left)))
            j = int(gen.integers(0, len(right)))
            events.append(("rank1", i, j, float(gen.normal(0.0, delta_sd))))
    return events


@dataclass
class StreamSpec:
    """stream.py:171-197: one synthetic run (matrix, events, policy, logging)."""

    m: int = 50
    n: int = 40
    true_rank: int = 5
    noise_scale: float = 0.05
    k: int = 5
    seed: int = 0
    scenario: str = "rank1"  # rank1 | rows | cols | mixed
    events: int = 10_000
    delta_sd: float = 0.05
    mix_weights: tuple = (0.05, 0.05, 0.90)
    policy: object = None
    log_every: int = 50
    tol: float = 1e-10
    reortho_guard: bool = False

    def __post_init__(self):
        if self.scenario not in ("rank1", "rows", "cols", "mixed"):
            raise ValueError(f"unknown scenario {self.scenario!r}")
        if self.events < 0:
            raise ValueError(f"events must be >= 0, got {self.events}")
        if self.log_every < 1:
            raise ValueError(f"log_every must be >= 1, got {self.log_every}")
        if self.policy is None:
            from .policies import PolicyConfig

            self.policy = PolicyConfig()


def build_events(spec: StreamSpec):
    """stream.py:200-220."""
    if spec.scenario == "rank1":
        return gen_rank_one_events(spec.events, spec.delta_sd, spec.m, spec.n, spec.seed)
    if spec.scenario == "rows":
        return gen_structural_events("row", spec.events, spec.true_rank, spec.noise_scale,
                                     spec.n, spec.seed)
    if spec.scenario == "cols":
        return gen_structural_events("col", spec.events, spec.true_rank, spec.noise_scale,
                                     spec.m, spec.seed)
    return gen_mixed_stream(spec.events, spec.mix_weights, spec.m, spec.n, spec.true_rank,
                            spec.noise_scale, spec.delta_sd, spec.seed)


def run_simulation(spec: StreamSpec, return_engine: bool = False):
    """stream.py:257-333 on the device engine: the spec's generated matrix and
    events through stream.run_stream (Algorithm 1)."""
    from .stream import run_stream

    initial = gen_low_rank(spec.m, spec.n, spec.true_rank, spec.noise_scale, spec.seed)
    return run_stream(initial, to_stream_events(build_events(spec)), spec.k, spec.policy,
                      log_every=spec.log_every, tol=spec.tol, reortho_guard=spec.reortho_guard,
                      return_engine=return_engine)

"""Event types and the Algorithm-1 simulation loop (mirror of svdstream/stream.py).

``run_stream`` is ``run_simulation`` (stream.py:257-333) with the initial
matrix and the event list passed in explicitly; ``workloads.run_simulation``
drives it from a ``StreamSpec`` with the reference's own generators, and
BASELINE's seeded inputs come from ``workloads.cfg1..cfg5a``.
"""

from __future__ import annotations

import time
from dataclasses import dataclass

import numpy as np

from .engine import SvdEngine
from .metrics import (MetricsRecord, OracleResult, angle_to_opt, collect, compute_oracle,
                      error_ratio, frob_error)
from .policies import (PolicyConfig, angle_should_refresh, error_should_refresh, evr_select_rank,
                       novelty_rank_bump, periodic_should_refresh)


@dataclass(frozen=True)
class RowAppend:
    values: np.ndarray


@dataclass(frozen=True)
class ColAppend:
    values: np.ndarray


@dataclass(frozen=True)
class RankOneUpdate:
    i: int
    j: int
    delta: float


UpdateEvent = RowAppend | ColAppend | RankOneUpdate


def apply_event(engine: SvdEngine, event) -> None:
    """Dispatch one event to the engine (stream.py:59-68)."""
    if isinstance(event, RowAppend):
        engine.row_append(event.values)
    elif isinstance(event, ColAppend):
        engine.col_append(event.values)
    elif isinstance(event, RankOneUpdate):
        engine.rank_one_update(event.i, event.j, event.delta)
    else:
        raise TypeError(f"unknown event type {type(event).__name__}")


class _AdaptiveRankState:
    """Hysteresis for energy-based rank selection (stream.py:227-254)."""

    def __init__(self, config):
        self.config = config
        self.pending: int | None = None
        self.armed: int | None = None

    def observe(self, spectrum, current_k: int) -> None:
        cfg = self.config
        selected = evr_select_rank(spectrum, cfg.tau, cfg.k_min, cfg.k_max)
        if selected == current_k:
            self.pending = None
            self.armed = None
        elif selected == self.pending:
            self.armed = selected
        else:
            self.pending = selected
            self.armed = None

    def take_armed(self) -> int | None:
        armed, self.armed, self.pending = self.armed, None, None
        return armed


def run_stream(initial, events, k: int, policy: PolicyConfig | None = None,
               log_every: int = 50, tol: float = 1e-10, reortho_guard: bool = False,
               return_engine: bool = False):
    """Algorithm 1 (stream.py:257-333): one MetricsRecord per logical step."""
    policy = policy or PolicyConfig()
    if log_every < 1:
        raise ValueError(f"log_every must be >= 1, got {log_every}")
    start = time.perf_counter()
    engine = SvdEngine(initial, k, tol=tol, reortho_guard=reortho_guard)
    init_time = time.perf_counter() - start
    engine.set_reference()
    adaptive = _AdaptiveRankState(policy.adaptive) if policy.adaptive else None
    records: list[MetricsRecord] = [
        collect(engine, update_time=init_time, refreshed=False,
                oracle=compute_oracle(engine, engine.work_rank))
    ]
    t_last_refresh = 0
    for t, event in enumerate(events, start=1):
        start = time.perf_counter()
        try:
            apply_event(engine, event)
        except ValueError as exc:
            raise ValueError(f"event at step {t} failed: {exc}") from exc
        engine.synchronize()  # the update is complete when its kernels are (stream.py:284-289)
        update_time = time.perf_counter() - start

        if adaptive and isinstance(event, (RowAppend, ColAppend)):
            bumped = novelty_rank_bump(engine.last_residual, engine.last_input_norm,
                                       policy.adaptive.eta, engine.work_rank,
                                       policy.adaptive.k_max)
            if bumped != engine.work_rank:
                engine.set_rank(bumped)

        oracle: OracleResult | None = None
        if t % log_every == 0:
            oracle = compute_oracle(engine, engine.work_rank)
            if adaptive:
                adaptive.observe(oracle.singular_values, engine.work_rank)

        fire = False
        if policy.kind == "periodic":
            fire = periodic_should_refresh(t, policy.period)
        elif policy.kind == "error" and oracle is not None:
            fire = error_should_refresh(error_ratio(frob_error(engine), oracle.frob_opt),
                                        policy.gamma, t, t_last_refresh, policy.min_spacing)
        elif policy.kind == "angle" and oracle is not None:
            fire = angle_should_refresh(angle_to_opt(engine, oracle.basis), policy.theta_max)

        if fire:
            if adaptive:
                armed = adaptive.take_armed()
                if armed is not None:
                    engine.set_rank(armed)
            engine.refresh(store_reference=True)
            t_last_refresh = t

        records.append(collect(engine, update_time=update_time, refreshed=fire, oracle=oracle))
    if return_engine:
        return records, engine
    return records

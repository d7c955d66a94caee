"""Shared test configuration.

Markers:
  gpu -- needs a CUDA device (run on the B200 box with ``-m gpu``).
Everything unmarked runs on CPU in a few minutes.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

GOLDEN = ROOT / "tests" / "golden" / "reference_golden.npz"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: test needs a CUDA device (B200)")


@pytest.fixture(scope="session")
def golden():
    return np.load(GOLDEN)


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.fail("GPU test collected without a CUDA device")
    return torch.device("cuda:0")


def rel_err(a, b, floor=1e-300):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), floor))) if a.size else 0.0


def sine_angle(q1, q2):
    """Largest principal angle via asin(||(I - Q1 Q1^T) Q2||_2) (parity metric)."""
    q1 = np.asarray(q1)
    q2 = np.asarray(q2)
    r = q2 - q1 @ (q1.T @ q2)
    return float(np.arcsin(min(1.0, np.linalg.norm(r, 2)))) if r.size else 0.0


# --------------------------------------------------- reference trajectories
# tests/golden/make_golden.py runs whole BASELINE streams through the
# reference's own loop (svdstream.stream.run_simulation) and stores one row
# per MetricsRecord: step, frob_error, evr, rank, refreshed, frob_opt,
# frob_ratio, angle_ref, angle_opt (None -> NaN).
SIM_TRAJ_RTOL = 1e-8  # north_star: metric trajectories within 1e-8 relative
SIM_ANGLE_ATOL = 1e-6  # north_star: principal angles below 1e-6 rad


def sim_array(records):
    nan = lambda v: np.nan if v is None else float(v)
    return np.array([[r.step, r.frob_error, r.evr, r.rank, float(r.refreshed), nan(r.frob_opt),
                      nan(r.frob_ratio), nan(r.angle_ref), nan(r.angle_opt)] for r in records])


def check_sim(golden, tag, got, n=None):
    """Compare a trajectory (prefix of length n) with the reference's."""
    ref = golden[f"sim_{tag}_records"]
    if n is not None:
        ref = ref[:n]
    assert got.shape == ref.shape, (got.shape, ref.shape)
    # step, rank and refresh flags exactly
    np.testing.assert_array_equal(got[:, [0, 3, 4]], ref[:, [0, 3, 4]])
    for c in (1, 2, 5, 6):  # frob_error, evr, frob_opt, frob_ratio
        ok = ~np.isnan(ref[:, c])
        np.testing.assert_array_equal(np.isnan(got[:, c]), ~ok, err_msg=f"column {c} NaN pattern")
        np.testing.assert_allclose(got[ok, c], ref[ok, c], rtol=SIM_TRAJ_RTOL, atol=1e-300,
                                   err_msg=f"column {c}")
    for c in (7, 8):  # angle_ref, angle_opt (arccos-based, as the reference)
        ok = ~np.isnan(ref[:, c])
        np.testing.assert_array_equal(np.isnan(got[:, c]), ~ok, err_msg=f"column {c} NaN pattern")
        if ok.any():
            assert np.max(np.abs(got[ok, c] - ref[ok, c])) < SIM_ANGLE_ATOL, f"column {c}"


def decode_events(kinds, vecs, m, n):
    """Inverse of make_golden._encode_events."""
    ev, off = [], 0
    for k, i, j, d in kinds:
        if k == 0:
            ev.append(("row", vecs[off:off + n]))
            off += n
            m += 1
        elif k == 1:
            ev.append(("col", vecs[off:off + m]))
            off += m
            n += 1
        else:
            ev.append(("rank1", int(i), int(j), float(d)))
    return ev


def sim_inputs(golden, tag):
    """(a0, events, k, policy kwargs, log_every) of a stored reference run,
    regenerated from the same seeded workloads as make_golden.py."""
    from paper_2605_24514_b200 import workloads

    if tag == "cfg1":
        a0, ev, _ = workloads.cfg1(0, n_events=1000)
        return a0, ev, 10, dict(kind="periodic", period=100), 1
    if tag == "cfg2":
        a0, ev, _ = workloads.cfg2(0, n_events=2000)
        return a0, ev, 20, dict(kind="error", gamma=1.05, min_spacing=0), 1
    if tag == "cfg3":
        a0, ev, _ = workloads.cfg3(0)
        return a0, ev, 5, dict(kind="angle", theta_max=float(np.deg2rad(5.0))), 1
    if tag in ("cfg4r", "cfg4b"):
        a0, ev, _ = workloads.cfg4(0, m=400, n=120, rank=64, n_blocks=200)
        if tag == "cfg4r":
            return a0, ev, 64, dict(kind="periodic", period=200,
                                    adaptive=dict(tau=0.95, k_min=1, k_max=128, eta=0.5)), 50
        return a0, ev[:600], 12, dict(kind="periodic", period=150,
                                      adaptive=dict(tau=0.99, k_min=4, k_max=40, eta=0.05)), 25
    if tag == "guard":
        a0 = golden["sim_guard_a0"]
        ev = decode_events(golden["sim_guard_kinds"], golden["sim_guard_vecs"], *a0.shape)
        return a0, ev, 6, dict(kind="periodic", period=80), 10
    raise KeyError(tag)


# ----------------------------------------------------- reference CSV files
GOLDEN_DIR = ROOT / "tests" / "golden"


def read_table(path):
    """(header lines, column names, rows as lists of strings) of a file in
    the reference's record format (cli.py:74-83), plain or gzipped."""
    import gzip

    p = Path(path)
    text = gzip.open(p, "rt").read() if p.suffix == ".gz" else p.read_text()
    lines = text.splitlines()
    cols = lines[2].split(",")
    return lines[:2], cols, [ln.split(",") for ln in lines[3:]]


def compare_tables(ours, ref, *, exact=(), angles=(), skip=("update_time", "opt_time"),
                   rtol=1e-8, floors=None):
    """Column-by-column diff of two record files: `exact` columns equal as
    text, `angles` (arccos-based, ill-conditioned near 0) within 1e-6 rad or
    1e-11 in cosine, every other column within rtol relative (NaN where the
    reference has NaN) plus an absolute floor for differences of nearly
    equal operands: floors = {column: (atol, scale column or None)} allows
    |d| <= atol * |scale| (e.g. frob_gap = frob_error - frob_opt is zero up to
    rounding of its operands right after a refresh; a risk_rel_error of 1e-8
    is a difference of two volatilities that agree to 1e-11 relative)."""
    floors = floors or {}
    _, c1, r1 = read_table(ours)
    _, c2, r2 = read_table(ref)
    assert c1 == c2, (c1, c2)
    assert len(r1) == len(r2), (len(r1), len(r2))
    for j, name in enumerate(c1):
        if name in skip:
            continue
        a = [row[j] for row in r1]
        b = [row[j] for row in r2]
        if name in exact:
            assert a == b, f"column {name} differs"
            continue
        x = np.array([float(v) for v in a])
        y = np.array([float(v) for v in b])
        assert np.array_equal(np.isnan(x), np.isnan(y)), f"column {name}: NaN pattern"
        ok = ~np.isnan(y)
        if name in angles:
            bad = (np.abs(x[ok] - y[ok]) > 1e-6) & (np.abs(np.cos(x[ok]) - np.cos(y[ok])) > 1e-11)
            assert not bad.any(), f"column {name}: {np.max(np.abs(x[ok] - y[ok]))}"
        else:
            tol = rtol * np.abs(y[ok])
            if name in floors:
                atol, scale = floors[name]
                sc = (np.abs(np.array([float(row[c1.index(scale)]) for row in r2]))[ok]
                      if scale else 1.0)
                tol = tol + atol * sc
            bad = np.abs(x[ok] - y[ok]) > tol
            assert not bad.any(), (f"column {name}: max |d| {np.max(np.abs(x[ok] - y[ok]))}, "
                                   f"{int(bad.sum())} of {int(ok.sum())} rows")

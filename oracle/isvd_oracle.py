"""Numpy restatement of the reference incremental-SVD path — TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
leg may import this module.  It is the *checker*, never the product.

Every function cites the reference code it restates.  Paths are relative to
``/root/reference/pkg/src/svdstream/`` unless stated otherwise.  The
restatement is pinned against outputs of the real reference committed under
``tests/golden/`` (see ``tests/test_oracle_golden.py``).

Two small-core SVD flavours are restated, exactly as the reference has two
kernel backends (``backend.py:28``):

* ``core_svd_lapack``  -- ``_kernels_py.py:14-19`` (LAPACK gesdd via numpy)
* ``core_svd_jacobi``  -- ``_kernels.pyx:22-109`` (cyclic one-sided Jacobi)
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

# linalg.py:18 -- relative cutoff under which a singular value is reported 0
ZERO_SV_RTOL = 1e-12
# _kernels.pyx:17-19 -- Jacobi orthogonality target and sweep cap
ORTHO_EPS = 1e-14
MAX_SWEEPS = 64
# engine.py:30 -- defect beyond which the optional guard re-factors
REORTHO_THRESHOLD = 1e-6
# metrics.py:25 -- ratio denominators below this relative floor are "zero"
RATIO_FLOOR = 1e-12

__all__ = [
    "ZERO_SV_RTOL", "ORTHO_EPS", "MAX_SWEEPS", "REORTHO_THRESHOLD", "RATIO_FLOOR",
    "Factors", "as_matrix", "as_vector", "canonicalize_signs", "snap_small",
    "full_svd", "truncated_svd", "reconstruct", "orthonormality_defect",
    "principal_angle_max", "sine_angle_max", "core_svd_lapack", "core_svd_jacobi",
    "kernel_row_append", "kernel_rank_one", "OracleEngine", "OracleResult",
    "Record", "compute_oracle", "frob_error", "error_ratio", "evr",
    "angle_to_ref", "angle_to_opt", "collect", "PolicyConfig",
    "AdaptiveRankConfig", "periodic_should_refresh", "error_should_refresh",
    "angle_should_refresh", "evr_select_rank", "novelty_rank_bump",
    "AdaptiveRankState", "run_stream", "low_rank_covariance",
    "covariance_rel_error", "portfolio_vol", "risk_rel_error",
]


# --------------------------------------------------------------- linalg.py


def as_matrix(a, name: str = "matrix") -> np.ndarray:
    """linalg.py:21-28: 2-D, finite, C-contiguous float64."""
    arr = np.asarray(a, dtype=np.float64)
    if arr.ndim != 2:
        raise ValueError(f"{name} must be 2-D, got shape {arr.shape}")
    if not np.isfinite(arr).all():
        raise ValueError(f"{name} contains non-finite entries")
    return np.ascontiguousarray(arr)


def as_vector(x, length: int | None = None, name: str = "vector") -> np.ndarray:
    """linalg.py:31-40: 1-D, optional length, finite, C-contiguous float64."""
    vec = np.asarray(x, dtype=np.float64)
    if vec.ndim != 1:
        raise ValueError(f"{name} must be 1-D, got shape {vec.shape}")
    if length is not None and vec.shape[0] != length:
        raise ValueError(f"{name} has length {vec.shape[0]}, expected {length}")
    if not np.isfinite(vec).all():
        raise ValueError(f"{name} contains non-finite entries")
    return np.ascontiguousarray(vec)


@dataclass
class Factors:
    """linalg.py:43-60 (SvdFactors): u (m, r), s (r,), vt (r, n)."""

    u: np.ndarray
    s: np.ndarray
    vt: np.ndarray

    @property
    def rank(self) -> int:
        return int(self.s.shape[0])

    def copy(self) -> "Factors":
        return Factors(self.u.copy(), self.s.copy(), self.vt.copy())


def canonicalize_signs(u: np.ndarray, vt: np.ndarray) -> None:
    """linalg.py:63-75: make each U column's largest-|entry| (first on ties)
    nonnegative, negating the paired Vt row."""
    if u.shape[1] == 0:
        return
    lead = np.abs(u).argmax(axis=0)
    neg = u[lead, np.arange(u.shape[1])] < 0.0
    if neg.any():
        u[:, neg] = -u[:, neg]
        vt[neg, :] = -vt[neg, :]


def snap_small(s: np.ndarray) -> np.ndarray:
    """linalg.py:78-81: values below ZERO_SV_RTOL * s[0] become exactly 0."""
    if s.size and s[0] > 0.0:
        s[s < ZERO_SV_RTOL * s[0]] = 0.0
    return s


def full_svd(a) -> Factors:
    """linalg.py:84-92: thin LAPACK SVD, snapped, sign-canonical."""
    mat = as_matrix(a)
    u, s, vt = np.linalg.svd(mat, full_matrices=False)
    u = np.ascontiguousarray(u)
    vt = np.ascontiguousarray(vt)
    snap_small(s)
    canonicalize_signs(u, vt)
    return Factors(u, s, vt)


def truncated_svd(a, k: int) -> Factors:
    """linalg.py:95-109: top min(k, m, n) triplets (exact zeros kept)."""
    if k < 1:
        raise ValueError(f"k must be >= 1, got {k}")
    f = full_svd(a)
    w = min(int(k), f.rank)
    return Factors(np.ascontiguousarray(f.u[:, :w]), f.s[:w].copy(),
                   np.ascontiguousarray(f.vt[:w, :]))


def reconstruct(f: Factors) -> np.ndarray:
    """linalg.py:112-118: u @ diag(s) @ vt."""
    if f.u.shape[1] != f.s.shape[0] or f.vt.shape[0] != f.s.shape[0]:
        raise ValueError("inconsistent factor shapes")
    return (f.u * f.s) @ f.vt


def orthonormality_defect(q) -> float:
    """linalg.py:126-130: ||q^T q - I||_F."""
    q = np.asarray(q, dtype=np.float64)
    return float(np.linalg.norm(q.T @ q - np.eye(q.shape[1])))


def principal_angle_max(q1, q2) -> float:
    """linalg.py:133-153: arccos of the smallest singular value of q1^T q2."""
    q1 = as_matrix(q1, "q1")
    q2 = as_matrix(q2, "q2")
    if q1.shape[0] != q2.shape[0]:
        raise ValueError("ambient dimensions differ")
    if q1.shape[1] != q2.shape[1]:
        raise ValueError("column counts differ")
    if q1.shape[1] == 0:
        raise ValueError("subspaces must have at least one column")
    for name, q in (("q1", q1), ("q2", q2)):
        if orthonormality_defect(q) > 1e-6:
            raise ValueError(f"{name} is not orthonormal (defect > 1e-6)")
    sv = np.linalg.svd(q1.T @ q2, compute_uv=False)
    return float(np.arccos(min(1.0, max(0.0, float(sv[-1])))))


def sine_angle_max(q1, q2) -> float:
    """Largest principal angle via asin(||(I - Q1 Q1^T) Q2||_2).

    Not in the reference: the parity tests use it because the reference's
    arccos form floors at ~1e-8 rad (hard part 4)."""
    q1 = np.asarray(q1, dtype=np.float64)
    q2 = np.asarray(q2, dtype=np.float64)
    resid = q2 - q1 @ (q1.T @ q2)
    return float(np.arcsin(min(1.0, np.linalg.norm(resid, 2))))


# ------------------------------------------------ _kernels_py / _kernels.pyx


def core_svd_lapack(core):
    """_kernels_py.py:14-19: LAPACK SVD of the small core, snapped."""
    u, s, vt = np.linalg.svd(np.asarray(core, dtype=np.float64))
    snap_small(s)
    return u, s, vt


def _jacobi_sweeps(g: np.ndarray, v: np.ndarray) -> int:
    """_kernels.pyx:22-59: cyclic-by-rows one-sided Jacobi on columns of g,
    accumulating the same rotations into v.  Returns the sweeps used."""
    n = g.shape[0]
    for sweep in range(MAX_SWEEPS):
        rotated = False
        for p in range(n - 1):
            for q in range(p + 1, n):
                gp = g[:, p]
                gq = g[:, q]
                app = float(gp @ gp)
                aqq = float(gq @ gq)
                apq = float(gp @ gq)
                if abs(apq) <= ORTHO_EPS * math.sqrt(app * aqq):
                    continue
                rotated = True
                zeta = (aqq - app) / (2.0 * apq)
                if zeta >= 0.0:
                    t = 1.0 / (zeta + math.sqrt(1.0 + zeta * zeta))
                else:
                    t = -1.0 / (-zeta + math.sqrt(1.0 + zeta * zeta))
                c = 1.0 / math.sqrt(1.0 + t * t)
                sn = t * c
                g[:, p], g[:, q] = c * gp - sn * gq, sn * gp + c * gq
                vp = v[:, p].copy()
                vq = v[:, q].copy()
                v[:, p] = c * vp - sn * vq
                v[:, q] = sn * vp + c * vq
        if not rotated:
            return sweep + 1
    return MAX_SWEEPS


def _complete_basis_std(u: np.ndarray, cols) -> None:
    """_kernels.pyx:62-79: fill listed columns with the first standard basis
    vector whose component orthogonal to the other columns has norm > 0.5."""
    m = u.shape[0]
    for j in cols:
        others = [c for c in range(u.shape[1]) if c != j]
        basis = u[:, others]
        for axis in range(m):
            cand = np.zeros(m)
            cand[axis] = 1.0
            cand -= basis @ (basis.T @ cand)
            nrm = float(np.linalg.norm(cand))
            if nrm > 0.5:
                u[:, j] = cand / nrm
                break
        else:
            raise ValueError("cannot complete an orthonormal basis")


def core_svd_jacobi(core):
    """_kernels.pyx:82-109: Jacobi SVD, stable descending sort, snap, divide
    the surviving columns by their raw norms, complete the dead ones."""
    a = np.array(core, dtype=np.float64)
    if a.ndim != 2 or a.shape[0] != a.shape[1]:
        raise ValueError(f"core must be square, got shape {a.shape}")
    n = a.shape[0]
    g = a.copy()
    v = np.eye(n)
    _jacobi_sweeps(g, v)
    raw = np.sqrt((g * g).sum(axis=0))
    order = np.argsort(-raw, kind="stable")
    raw = raw[order]
    g = g[:, order]
    v = v[:, order]
    s = raw.copy()
    if n and s[0] > 0.0:
        s[s < ZERO_SV_RTOL * s[0]] = 0.0
    u = np.zeros((n, n))
    live = s > 0.0
    u[:, live] = g[:, live] / raw[live]
    dead = np.flatnonzero(~live)
    if dead.size:
        _complete_basis_std(u, dead)
    return u, s, np.ascontiguousarray(v.T)


def kernel_row_append(u, s, vt, x, tol, keep, core_svd=core_svd_lapack):
    """_kernels_py.py:22-49 / _kernels.pyx:112-187: Brand row append.

    p = Vt x; z = x - Vt^T p (one classical Gram-Schmidt pass); rho = ||z||;
    core [[diag s, 0], [p, rho]] (rho and the injected direction zeroed when
    rho <= tol); U' = [U 0; 0 1] Uk[:, :keep]; Vt' = Vk^T[:keep, :r] Vt +
    Vk^T[:keep, r] (x) z_hat.  Returns (u', s', vt', rho)."""
    m, r = u.shape
    n = vt.shape[1]
    proj = vt @ x
    resid = x - vt.T @ proj
    rho = float(np.linalg.norm(resid))
    core = np.zeros((r + 1, r + 1))
    core[np.arange(r), np.arange(r)] = s
    core[r, :r] = proj
    if rho > tol:
        core[r, r] = rho
        inject = resid / rho
    else:
        inject = np.zeros(n)
    uk, s_new, vkt = core_svd(core)
    u_new = np.empty((m + 1, keep))
    u_new[:m] = u @ uk[:r, :keep]
    u_new[m] = uk[r, :keep]
    vt_new = vkt[:keep, :r] @ vt + np.outer(vkt[:keep, r], inject)
    return u_new, s_new[:keep].copy(), vt_new, rho


def kernel_rank_one(u, s, vt, i, j, delta, keep, core_svd=core_svd_lapack):
    """_kernels_py.py:52-58 / _kernels.pyx:190-237: projection rule
    K = diag(s) + delta * U[i,:]^T Vt[:,j]^T; U' = U Uk; Vt' = Vk^T Vt."""
    core = np.diag(s) + delta * np.outer(u[i, :], vt[:, j])
    uk, s_new, vkt = core_svd(core)
    return u @ uk[:, :keep], s_new[:keep].copy(), vkt[:keep, :] @ vt


# --------------------------------------------------------------- engine.py


def _orthonormal_completion(q: np.ndarray, j: int) -> None:
    """engine.py:33-56: replace column j by a unit vector orthogonal to the
    other columns -- first its own direction, then e_0, e_1, ..."""
    m, w = q.shape
    others = [c for c in range(w) if c != j]
    basis = q[:, others]
    col = q[:, j].copy()
    col -= basis @ (basis.T @ col)
    nrm = float(np.linalg.norm(col))
    if nrm > 0.5:
        q[:, j] = col / nrm
        return
    for axis in range(m):
        cand = np.zeros(m)
        cand[axis] = 1.0
        cand -= basis @ (basis.T @ cand)
        nrm = float(np.linalg.norm(cand))
        if nrm > 0.5:
            q[:, j] = cand / nrm
            return
    raise ValueError("cannot complete an orthonormal basis: width exceeds dimension")


def _complete_zero_columns(u: np.ndarray, vt: np.ndarray, s: np.ndarray) -> None:
    """engine.py:59-70: for every exact-zero singular value, repair the U
    column and then the V column whose squared norm is off by > 1e-6."""
    for j in np.flatnonzero(s == 0.0):
        for q in (u, vt.T):
            nsq = float(q[:, j] @ q[:, j])
            if abs(nsq - 1.0) > 1e-6:
                _orthonormal_completion(q, j)


class OracleEngine:
    """engine.py:73-217 (SvdEngine) restated: dense tracked matrix, squared
    norm recurrences, factor install (completion, guard, signs)."""

    def __init__(self, a0, k: int, tol: float = 1e-10, reortho_guard: bool = False,
                 core_svd=core_svd_lapack):
        a0 = as_matrix(a0, "initial matrix")
        if a0.size == 0:
            raise ValueError("initial matrix must be nonempty")
        if k < 1:
            raise ValueError(f"work rank must be >= 1, got {k}")
        if not tol > 0.0:
            raise ValueError(f"tol must be positive, got {tol}")
        self.work_rank = int(k)
        self.tol = float(tol)
        self.reortho_guard = bool(reortho_guard)
        self.core_svd = core_svd
        self._tracked = a0.copy()
        self._sq_norm = float(np.sum(a0 * a0))
        self.factors = truncated_svd(a0, self.work_rank)
        self.step = 0
        self.ref_subspace = None
        self.last_residual = float("nan")
        self.last_input_norm = float("nan")

    @property
    def shape(self):
        return tuple(self._tracked.shape)

    @property
    def tracked(self):
        return self._tracked

    @property
    def sq_norm(self):
        return self._sq_norm

    def tracked_sq_norm(self):
        return self._sq_norm

    def row_append(self, x) -> None:
        """engine.py:117-129."""
        m, n = self._tracked.shape
        x = as_vector(x, length=n, name="appended row")
        f = self.factors
        keep = min(f.rank + 1, self.work_rank, m + 1, n)
        u, s, vt, rho = kernel_row_append(f.u, f.s, f.vt, x, self.tol, keep, self.core_svd)
        self.last_input_norm = float(np.linalg.norm(x))
        self.last_residual = rho
        self._install(u, s, vt)
        self._tracked = np.vstack([self._tracked, x[None, :]])
        self._sq_norm += float(x @ x)
        self.step += 1

    def col_append(self, y) -> None:
        """engine.py:131-147 (transpose trick)."""
        m, n = self._tracked.shape
        y = as_vector(y, length=m, name="appended column")
        f = self.factors
        keep = min(f.rank + 1, self.work_rank, m, n + 1)
        ut = np.ascontiguousarray(f.vt.T)
        vtt = np.ascontiguousarray(f.u.T)
        ut2, s, vtt2, rho = kernel_row_append(ut, f.s, vtt, y, self.tol, keep, self.core_svd)
        self.last_input_norm = float(np.linalg.norm(y))
        self.last_residual = rho
        self._install(np.ascontiguousarray(vtt2.T), s, np.ascontiguousarray(ut2.T))
        self._tracked = np.hstack([self._tracked, y[:, None]])
        self._sq_norm += float(y @ y)
        self.step += 1

    def rank_one_update(self, i: int, j: int, delta: float) -> None:
        """engine.py:149-167."""
        m, n = self._tracked.shape
        if not (0 <= i < m and 0 <= j < n):
            raise ValueError(f"index ({i}, {j}) out of bounds for shape ({m}, {n})")
        delta = float(delta)
        if not np.isfinite(delta):
            raise ValueError("delta must be finite")
        f = self.factors
        u, s, vt = kernel_rank_one(f.u, f.s, f.vt, int(i), int(j), delta, f.rank,
                                   self.core_svd)
        self._install(u, s, vt)
        old = float(self._tracked[i, j])
        self._tracked[i, j] = old + delta
        self._sq_norm += 2.0 * delta * old + delta * delta
        self.step += 1

    def refresh(self, store_reference: bool = False) -> None:
        """engine.py:171-176."""
        self.factors = truncated_svd(self._tracked, self.work_rank)
        self._sq_norm = float(np.sum(self._tracked * self._tracked))
        if store_reference:
            self.ref_subspace = self.factors.u.copy()

    def set_reference(self) -> None:
        """engine.py:178-180."""
        self.ref_subspace = self.factors.u.copy()

    def set_rank(self, k_new: int) -> None:
        """engine.py:182-198."""
        if k_new < 1:
            raise ValueError(f"work rank must be >= 1, got {k_new}")
        self.work_rank = int(k_new)
        f = self.factors
        if f.rank > k_new:
            self.factors = Factors(np.ascontiguousarray(f.u[:, :k_new]),
                                   f.s[:k_new].copy(),
                                   np.ascontiguousarray(f.vt[:k_new, :]))

    def _install(self, u, s, vt) -> None:
        """engine.py:202-208."""
        if np.any(s == 0.0):
            _complete_zero_columns(u, vt, s)
        if self.reortho_guard:
            u, s, vt = self._reortho_if_needed(u, s, vt)
        canonicalize_signs(u, vt)
        self.factors = Factors(u, s, vt)

    def _reortho_if_needed(self, u, s, vt):
        """engine.py:210-217."""
        defect = max(orthonormality_defect(u), orthonormality_defect(vt.T))
        if defect <= REORTHO_THRESHOLD:
            return u, s, vt
        qu, ru = np.linalg.qr(u)
        qv, rv = np.linalg.qr(vt.T)
        uk, s2, vkt = self.core_svd((ru * s) @ rv.T)
        return np.ascontiguousarray(qu @ uk), s2, np.ascontiguousarray(vkt @ qv.T)


# -------------------------------------------------------------- metrics.py


@dataclass
class OracleResult:
    """metrics.py:46-53."""

    frob_opt: float
    basis: np.ndarray
    singular_values: np.ndarray


@dataclass
class Record:
    """metrics.py:28-43 (MetricsRecord) minus the wall-clock fields."""

    step: int
    frob_error: float
    evr: float
    rank: int
    refreshed: bool
    frob_opt: float | None = None
    frob_gap: float | None = None
    frob_ratio: float | None = None
    angle_ref: float | None = None
    angle_opt: float | None = None


def compute_oracle(a, k: int) -> OracleResult:
    """metrics.py:56-64: full SVD, optimal rank-k error, leading basis."""
    f = full_svd(a)
    w = min(int(k), f.rank)
    tail = f.s[w:]
    return OracleResult(float(np.sqrt(np.sum(tail * tail))), f.u[:, :w].copy(), f.s.copy())


def frob_error(engine) -> float:
    """metrics.py:74-76."""
    return float(np.linalg.norm(engine.tracked - reconstruct(engine.factors)))


def error_ratio(e_inc: float, e_opt: float) -> float:
    """metrics.py:79-83."""
    if e_opt > RATIO_FLOOR * max(1.0, e_inc):
        return e_inc / e_opt
    return float("nan")


def evr(engine) -> float:
    """metrics.py:86-93."""
    sq = engine.sq_norm
    if sq <= 0.0:
        raise ValueError("explained variance is undefined for a zero matrix")
    s = engine.factors.s
    return min(1.0, max(0.0, float(np.sum(s * s)) / sq))


def angle_to_ref(engine):
    """metrics.py:96-113."""
    ref = engine.ref_subspace
    if ref is None:
        return None
    u = engine.factors.u
    if ref.shape != u.shape:
        return None
    return principal_angle_max(u, ref)


def angle_to_opt(engine, basis) -> float:
    """metrics.py:116-119."""
    u = engine.factors.u
    return principal_angle_max(u, basis[:, : u.shape[1]])


def collect(engine, refreshed: bool, oracle: OracleResult | None = None) -> Record:
    """metrics.py:122-145."""
    e_inc = frob_error(engine)
    rec = Record(step=engine.step, frob_error=e_inc,
                 evr=evr(engine) if engine.sq_norm > 0.0 else float("nan"),
                 rank=engine.factors.rank, refreshed=bool(refreshed))
    if oracle is not None:
        rec.frob_opt = oracle.frob_opt
        rec.frob_gap = e_inc - oracle.frob_opt
        rec.frob_ratio = error_ratio(e_inc, oracle.frob_opt)
        rec.angle_ref = angle_to_ref(engine)
        rec.angle_opt = angle_to_opt(engine, oracle.basis)
    return rec


# ------------------------------------------------------------- policies.py


@dataclass
class AdaptiveRankConfig:
    """policies.py:15-32."""

    tau: float = 0.95
    k_min: int = 1
    k_max: int = 64
    eta: float = 0.5


@dataclass
class PolicyConfig:
    """policies.py:35-56 (validation lives in the product's mirror)."""

    kind: str = "none"
    period: int = 1000
    gamma: float = 1.1
    min_spacing: int = 0
    theta_max: float = 0.5
    adaptive: AdaptiveRankConfig | None = None


def periodic_should_refresh(t: int, period: int) -> bool:
    """policies.py:59-63."""
    return t > 0 and t % period == 0


def error_should_refresh(ratio, gamma, t, t_last, min_spacing) -> bool:
    """policies.py:66-73."""
    if ratio is None or math.isnan(ratio):
        return False
    return ratio > gamma and (t - t_last) >= min_spacing


def angle_should_refresh(angle, theta_max) -> bool:
    """policies.py:76-80."""
    if angle is None or math.isnan(angle):
        return False
    return angle > theta_max


def evr_select_rank(singular_values, tau, k_min, k_max) -> int:
    """policies.py:83-110: smallest k in [k_min, k_max] reaching tau."""
    energy = np.asarray(singular_values, dtype=np.float64) ** 2
    total = float(sum(float(e) for e in energy))
    if total <= 0.0:
        return k_min
    running = 0.0
    cumulative = []
    for e in energy:
        running += float(e)
        cumulative.append(running)
    for k in range(k_min, k_max + 1):
        if cumulative[min(k, len(cumulative)) - 1] / total >= tau:
            return k
    return k_max


def novelty_rank_bump(z_norm, x_norm, eta, k, k_max) -> int:
    """policies.py:113-124."""
    if x_norm > 0.0 and z_norm > eta * x_norm:
        return min(k + 1, k_max)
    return k


class AdaptiveRankState:
    """stream.py:227-254: two consecutive equal selections arm a new rank."""

    def __init__(self, cfg: AdaptiveRankConfig):
        self.cfg = cfg
        self.pending = None
        self.armed = None

    def observe(self, spectrum, current_k: int) -> None:
        sel = evr_select_rank(spectrum, self.cfg.tau, self.cfg.k_min, self.cfg.k_max)
        if sel == current_k:
            self.pending = None
            self.armed = None
        elif sel == self.pending:
            self.armed = sel
        else:
            self.pending = sel
            self.armed = None

    def take_armed(self):
        armed, self.armed, self.pending = self.armed, None, None
        return armed


# ---------------------------------------------------------------- stream.py


def run_stream(engine, events, policy: PolicyConfig, log_every: int):
    """stream.py:257-333 (Algorithm 1) with an explicit event list.

    ``events`` items are ("row", x) | ("col", y) | ("rank1", i, j, delta).
    Returns the list of Records (init record first)."""
    adaptive = AdaptiveRankState(policy.adaptive) if policy.adaptive else None
    engine.set_reference()
    records = [collect(engine, False, compute_oracle(engine.tracked, engine.work_rank))]
    t_last = 0
    for t, ev in enumerate(events, start=1):
        kind = ev[0]
        if kind == "row":
            engine.row_append(ev[1])
        elif kind == "col":
            engine.col_append(ev[1])
        elif kind == "rank1":
            engine.rank_one_update(ev[1], ev[2], ev[3])
        else:
            raise TypeError(f"unknown event type {kind!r}")
        if adaptive and kind in ("row", "col"):
            bumped = novelty_rank_bump(engine.last_residual, engine.last_input_norm,
                                       policy.adaptive.eta, engine.work_rank,
                                       policy.adaptive.k_max)
            if bumped != engine.work_rank:
                engine.set_rank(bumped)
        oracle = None
        if t % log_every == 0:
            oracle = compute_oracle(engine.tracked, engine.work_rank)
            if adaptive:
                adaptive.observe(oracle.singular_values, engine.work_rank)
        fire = False
        if policy.kind == "periodic":
            fire = periodic_should_refresh(t, policy.period)
        elif policy.kind == "error" and oracle is not None:
            fire = error_should_refresh(error_ratio(frob_error(engine), oracle.frob_opt),
                                        policy.gamma, t, t_last, policy.min_spacing)
        elif policy.kind == "angle" and oracle is not None:
            fire = angle_should_refresh(angle_to_opt(engine, oracle.basis), policy.theta_max)
        if fire:
            if adaptive:
                armed = adaptive.take_armed()
                if armed is not None:
                    engine.set_rank(armed)
            engine.refresh(store_reference=True)
            t_last = t
        records.append(collect(engine, fire, oracle))
    return records


# --------------------------------------------------------------- finance.py


def low_rank_covariance(s, vt, t: int) -> np.ndarray:
    """finance.py:326-335: V diag(s^2) V^T / (t-1), symmetrised."""
    v = vt.T
    cov = (v * (s ** 2)) @ v.T / (t - 1.0)
    return 0.5 * (cov + cov.T)


def covariance_rel_error(inc, orc) -> float:
    """finance.py:338-347."""
    return float(np.linalg.norm(inc - orc) / np.linalg.norm(orc))


def portfolio_vol(cov, w) -> float:
    """finance.py:350-364."""
    quad = float(w @ cov @ w)
    if quad < -1e-10:
        raise ValueError("covariance is not PSD")
    return math.sqrt(max(0.0, quad))


def risk_rel_error(vol_inc: float, vol_orc: float) -> float:
    """finance.py:367-371."""
    return abs(vol_inc - vol_orc) / vol_orc

"""Incremental truncated SVD engine on the B200 (drop-in for svdstream.engine).

``SvdEngine`` keeps the reference API (engine.py:73-198): the factors, the
tracked dense matrix and its squared norm live in HBM and every event is a
short sequence of sm_100a kernels issued by libisvd (see csrc/engine.cu for
the launch sequence).  Host-side work is limited to argument validation --
done *before* anything is launched, so a rejected event leaves the state
unchanged exactly like the reference (tests/test_engine.py:88-95) -- and to
lazily materialised host copies for the read-only properties.

``BatchedSvdEngine`` drives B independent streams of identical shape with
one launch sequence per tick (the batched-stream workload, BASELINE config 5a).
"""

from __future__ import annotations

import ctypes as C
import weakref

import numpy as np

from . import _lib
from .linalg import SvdFactors, as_matrix, as_vector

# engine.py:30
REORTHO_THRESHOLD = 1e-6


def _destroy(lib, handle):
    lib.isvd_engine_destroy(handle)


class _Handle:
    """Owner of one isvd_engine* (B streams)."""

    def __init__(self, batch, m, n, k, tol, guard, m_cap=0, n_cap=0, k_cap=0, stream=None):
        lib = _lib.load()
        h = C.c_void_p()
        _lib.check(lib.isvd_engine_create(C.byref(h), int(batch), int(m), int(n), int(k),
                                          float(tol), int(bool(guard)), int(m_cap), int(n_cap),
                                          int(k_cap), stream))
        self.lib = lib
        self.h = h
        self._fin = weakref.finalize(self, _destroy, lib, h)

    def shape(self):
        b, m, n, r, k = (C.c_int() for _ in range(5))
        step = C.c_int64()
        _lib.check(self.lib.isvd_engine_shape(self.h, C.byref(b), C.byref(m), C.byref(n),
                                              C.byref(r), C.byref(k), C.byref(step)))
        return b.value, m.value, n.value, r.value, k.value, step.value

    def stream(self) -> int:
        return int(self.lib.isvd_engine_stream(self.h) or 0)

    def streams(self) -> list[int]:
        """Engine stream + stream groups (no join): every stream that may
        read a device-resident event payload."""
        cap = 16
        buf = (C.c_void_p * cap)()
        n = int(self.lib.isvd_engine_streams(self.h, buf, cap))
        return [int(buf[i] or 0) for i in range(min(n, cap))]


class _DeviceInputs:
    """Stream ordering and lifetime of device-resident (torch) event payloads.

    The engine reads a payload on its own stream (rank-1 triples are staged
    and bounds-checked there) and, for appended rows / columns, on its stream
    groups, which may run ahead of the caller.  Before an event the engine
    stream waits for the caller's current torch stream (the producer); after
    it the tensor is marked as in use on every engine stream
    (Tensor.record_stream), so the caching allocator cannot hand its memory
    out again while a group still reads it."""

    def __init__(self, handle: _Handle):
        self._h = handle
        self._st0 = handle.stream()  # fixed for the engine's lifetime (join is a no-op here)
        self._ext = {}
        self._device = None

    def _wrap(self, torch, s: int):
        ext = self._ext.get(s)
        if ext is None:
            ext = self._ext[s] = torch.cuda.ExternalStream(s, device=self._device)
        return ext

    def check(self, t, dtype_name: str, shape, name: str):
        import torch

        if tuple(t.shape) != tuple(shape):
            raise ValueError(f"{name} has shape {tuple(t.shape)}, expected {tuple(shape)}")
        want = getattr(torch, dtype_name)
        if t.dtype != want:
            raise ValueError(f"{name} must be {dtype_name}, got {t.dtype}")
        if self._device is None:
            self._device = torch.device("cuda", torch.cuda.current_device())
        if t.device != self._device:
            raise ValueError(f"{name} is on {t.device}, the engine runs on {self._device}")
        return t.contiguous()

    def before(self):
        import torch

        cur = torch.cuda.current_stream(self._device)
        if cur.cuda_stream != self._st0:
            self._wrap(torch, self._st0).wait_stream(cur)

    def after(self, *tensors):
        import torch

        for s in self._h.streams():
            ext = self._wrap(torch, s)
            for t in tensors:
                t.record_stream(ext)


class BatchedSvdEngine:
    """B independent incremental-SVD streams of identical shape.

    Events take one row / column / entry per stream: ``row_append(X)`` with
    X of shape (B, n), ``col_append(Y)`` with (B, m), ``rank_one_update(I,
    J, D)`` with three length-B vectors.  Inputs may be numpy arrays (host)
    or CUDA torch tensors (device, trusted: no finiteness check)."""

    def __init__(self, a0, k: int, tol: float = 1e-10, reortho_guard: bool = False, *,
                 m_cap: int = 0, n_cap: int = 0, k_cap: int = 0, stream=None):
        if k < 1:
            raise ValueError(f"work rank must be >= 1, got {k}")
        if not tol > 0.0:
            raise ValueError(f"tol must be positive, got {tol}")
        on_dev = _is_device(a0)
        if on_dev:
            if a0.dim() != 3:
                raise ValueError("a0 must be (B, m, n)")
            batch, m, n = (int(v) for v in a0.shape)
            src = a0.contiguous()
        else:
            src = np.ascontiguousarray(np.asarray(a0, dtype=np.float64))
            if src.ndim != 3:
                raise ValueError("a0 must be (B, m, n)")
            batch, m, n = src.shape
        if m * n == 0:
            raise ValueError("initial matrix must be nonempty")
        self._h = _Handle(batch, m, n, k, tol, reortho_guard, m_cap, n_cap, k_cap, stream)
        self.tol = float(tol)
        self.reortho_guard = bool(reortho_guard)
        self._dev = _DeviceInputs(self._h)
        if on_dev:
            src = self._dev.check(src, "float64", (batch, m, n), "a0")
            self._dev.before()
        _lib.check(self._h.lib.isvd_engine_init(self._h.h, _lib.vptr(src), int(on_dev)))

    # ------------------------------------------------------------ state
    @property
    def batch(self) -> int:
        return self._h.shape()[0]

    @property
    def shape(self) -> tuple[int, int]:
        _, m, n, *_ = self._h.shape()
        return (m, n)

    @property
    def rank(self) -> int:
        return self._h.shape()[3]

    @property
    def work_rank(self) -> int:
        return self._h.shape()[4]

    @property
    def step(self) -> int:
        return self._h.shape()[5]

    @property
    def cuda_stream(self) -> int:
        """cudaStream_t (as int) all of this engine's kernels launch on."""
        return self._h.stream()

    def scalars(self):
        """(sq_norm, last_residual, last_input_norm), each of shape (B,)."""
        b = self.batch
        sq, rho, xn = np.empty(b), np.empty(b), np.empty(b)
        _lib.check(self._h.lib.isvd_engine_get_scalars(self._h.h, _lib.dptr(sq), _lib.dptr(rho),
                                                       _lib.dptr(xn)))
        return sq, rho, xn

    def scalars_async(self, out, slot: int = 0) -> None:
        """Enqueue the step's (sq_norm, residual, input norm) into `out`
        (pinned host memory, 3 x B doubles) without waiting; pair with
        scalars_wait(slot).  A host loop that waits on step t after issuing
        step t+1 keeps the GPU busy while it validates and uploads inputs."""
        _lib.check(self._h.lib.isvd_engine_scalars_async(self._h.h, _lib.vptr(out), int(slot)))

    def scalars_wait(self, slot: int = 0) -> None:
        _lib.check(self._h.lib.isvd_engine_scalars_wait(self._h.h, int(slot)))

    def factors(self, b: int = 0) -> SvdFactors:
        _, m, n, r, _, _ = self._h.shape()
        u, s, v = np.empty((m, r)), np.empty(r), np.empty((n, r))
        _lib.check(self._h.lib.isvd_engine_get_factors(self._h.h, int(b), _lib.dptr(u),
                                                       _lib.dptr(s), _lib.dptr(v)))
        return SvdFactors(u, s, np.ascontiguousarray(v.T))

    def tracked(self, b: int = 0) -> np.ndarray:
        _, m, n, *_ = self._h.shape()
        a = np.empty((m, n))
        _lib.check(self._h.lib.isvd_engine_get_tracked(self._h.h, int(b), _lib.dptr(a)))
        return a

    def synchronize(self) -> None:
        _lib.check(self._h.lib.isvd_engine_synchronize(self._h.h))

    def flush(self) -> None:
        """Materialise deferred basis rotations now."""
        _lib.check(self._h.lib.isvd_engine_flush(self._h.h))

    def set_lazy(self, on: bool) -> None:
        """Deferred left-basis rotation on (default) or off (eager per event)."""
        _lib.check(self._h.lib.isvd_engine_set_lazy(self._h.h, int(bool(on))))

    def set_vdefer(self, mode: int) -> None:
        """Deferred right-basis rotation on rank-1 updates: 0 off, 1 auto
        (batches >= 64 streams, the default), 2 whenever supported."""
        _lib.check(self._h.lib.isvd_engine_set_vdefer(self._h.h, int(mode)))

    def snapshot(self) -> None:
        """Device-side checkpoint of the whole state (restore() returns to it)."""
        _lib.check(self._h.lib.isvd_engine_snapshot(self._h.h))

    def restore(self) -> None:
        _lib.check(self._h.lib.isvd_engine_restore(self._h.h))

    # ------------------------------------------------------------ events
    def row_append(self, x) -> None:
        b, m, n, *_ = self._h.shape()
        self._append(x, (b, n), "appended row", self._h.lib.isvd_engine_row_append)

    def col_append(self, y) -> None:
        b, m, n, *_ = self._h.shape()
        self._append(y, (b, m), "appended column", self._h.lib.isvd_engine_col_append)

    def _append(self, x, shape, name, fn) -> None:
        if _is_device(x):
            src = self._dev.check(x, "float64", shape, name)
            self._dev.before()
            _lib.check(fn(self._h.h, _lib.vptr(src), 1))
            self._dev.after(src)
            return
        src, _ = _event_array(x, shape, name)
        _lib.check(fn(self._h.h, _lib.vptr(src), 0))

    def rank_one_update(self, i, j, delta) -> None:
        """Device tensors (int64 i, j; float64 delta) are bounds- and
        finiteness-checked on the device: a rejected entry is applied as a
        no-op and the next synchronising call raises ValueError."""
        b = self.batch
        if _is_device(i):
            ii = self._dev.check(i, "int64", (b,), "row index")
            jj = self._dev.check(j, "int64", (b,), "column index")
            dd = self._dev.check(delta, "float64", (b,), "delta")
            self._dev.before()
            _lib.check(self._h.lib.isvd_engine_rank_one(self._h.h, _lib.vptr(ii), _lib.vptr(jj),
                                                        _lib.vptr(dd), 1))
            self._dev.after(ii, jj, dd)
            return
        ii = np.ascontiguousarray(np.asarray(i, dtype=np.int64).reshape(b))
        jj = np.ascontiguousarray(np.asarray(j, dtype=np.int64).reshape(b))
        dd = np.ascontiguousarray(np.asarray(delta, dtype=np.float64).reshape(b))
        _lib.check(self._h.lib.isvd_engine_rank_one(self._h.h, _lib.vptr(ii), _lib.vptr(jj),
                                                    _lib.vptr(dd), 0))

    def refresh(self, store_reference: bool = False) -> None:
        _lib.check(self._h.lib.isvd_engine_refresh(self._h.h, int(bool(store_reference))))

    def set_reference(self) -> None:
        _lib.check(self._h.lib.isvd_engine_set_reference(self._h.h))

    def set_rank(self, k_new: int) -> None:
        if k_new < 1:
            raise ValueError(f"work rank must be >= 1, got {k_new}")
        _lib.check(self._h.lib.isvd_engine_set_rank(self._h.h, int(k_new)))

    # ----------------------------------------------------------- metrics
    def frob_error(self) -> np.ndarray:
        out = np.empty(self.batch)
        _lib.check(self._h.lib.isvd_engine_frob_error(self._h.h, _lib.dptr(out)))
        return out

    def ortho_defect(self):
        du, dv = np.empty(self.batch), np.empty(self.batch)
        _lib.check(self._h.lib.isvd_engine_ortho_defect(self._h.h, _lib.dptr(du), _lib.dptr(dv)))
        return du, dv

    def angle_to_reference(self) -> np.ndarray:
        """Per-stream largest principal angle to the stored reference; NaN
        where the reference is absent or has another shape (reference: None)."""
        out = np.empty(self.batch)
        _lib.check(self._h.lib.isvd_engine_angle(self._h.h, 0, None, 0, 0, _lib.dptr(out)))
        out[out < 0] = np.nan
        return out

    def angle_to_basis(self, q) -> np.ndarray:
        """Per-stream largest principal angle to bases q (B, m, r)."""
        dev = _is_device(q)
        src = q.contiguous() if dev else np.ascontiguousarray(np.asarray(q, dtype=np.float64))
        out = np.empty(self.batch)
        _lib.check(self._h.lib.isvd_engine_angle(self._h.h, 1, _lib.vptr(src), int(src.shape[-1]),
                                                 int(dev), _lib.dptr(out)))
        return out

    def oracle(self, w_keep: int):
        """Device batch SVD of every tracked matrix: (s_all (B, nc), u (B, m, w))."""
        b, m, n, *_ = self._h.shape()
        nc = min(m, n)
        w = max(0, min(int(w_keep), nc))
        s = np.empty((b, nc))
        u = np.empty((b, m, w))
        _lib.check(self._h.lib.isvd_engine_oracle(self._h.h, w, _lib.dptr(s), _lib.dptr(u)))
        return s, u


def _is_device(x) -> bool:
    return hasattr(x, "is_cuda") and bool(x.is_cuda)


def _event_array(x, shape, name):
    arr = np.asarray(x, dtype=np.float64)
    if arr.shape != tuple(shape):
        raise ValueError(f"{name} has shape {arr.shape}, expected {shape}")
    # finiteness is checked by libisvd before any device work (ValueError)
    return np.ascontiguousarray(arr), 0


class SvdEngine:
    """Single-owner mutable state of one incremental SVD stream (engine.py:73).

    Same constructor, methods and properties as the reference; computation
    runs on the GPU.  ``factors``, ``tracked`` and ``ref_subspace`` are host
    copies materialised on access (cached until the next mutation);
    assigning ``factors`` / ``ref_subspace`` uploads new values."""

    def __init__(self, a0, k: int, tol: float = 1e-10, reortho_guard: bool = False, *,
                 capacity: tuple[int, int, int] | None = None, stream=None):
        a0 = as_matrix(a0, "initial matrix")
        if a0.size == 0:
            raise ValueError("initial matrix must be nonempty")
        if k < 1:
            raise ValueError(f"work rank must be >= 1, got {k}")
        if not tol > 0.0:
            raise ValueError(f"tol must be positive, got {tol}")
        m, n = a0.shape
        mc, nc, kc = capacity or (2 * m + 8, n, k)
        self._h = _Handle(1, m, n, k, tol, reortho_guard, mc, nc, kc, stream)
        self.tol = float(tol)
        self.reortho_guard = bool(reortho_guard)
        # the module constant is read when the engine is built, so a test can
        # force the guard the way the reference's does (monkeypatching
        # engine.REORTHO_THRESHOLD, tests/test_engine.py:309-323)
        self.reortho_threshold = REORTHO_THRESHOLD
        _lib.check(self._h.lib.isvd_engine_init(self._h.h, _lib.dptr(a0), 0))
        self._version = 0
        self._cache: dict = {}

    # ------------------------------------------------------------- views
    def _touch(self):
        self._version += 1
        self._cache.clear()

    def synchronize(self) -> None:
        """Wait for this engine's queued device work (events are asynchronous)."""
        _lib.check(self._h.lib.isvd_engine_synchronize(self._h.h))

    def _shape_all(self):
        return self._h.shape()

    @property
    def shape(self) -> tuple[int, int]:
        _, m, n, *_ = self._shape_all()
        return (m, n)

    @property
    def step(self) -> int:
        return self._shape_all()[5]

    @property
    def work_rank(self) -> int:
        return self._shape_all()[4]

    @property
    def tracked(self) -> np.ndarray:
        """The exact current matrix (host copy; do not mutate)."""
        if "tracked" not in self._cache:
            _, m, n, *_ = self._shape_all()
            a = np.empty((m, n))
            _lib.check(self._h.lib.isvd_engine_get_tracked(self._h.h, 0, _lib.dptr(a)))
            a.flags.writeable = False
            self._cache["tracked"] = a
        return self._cache["tracked"]

    def _scalars(self):
        if "scalars" not in self._cache:
            sq, rho, xn = np.empty(1), np.empty(1), np.empty(1)
            _lib.check(self._h.lib.isvd_engine_get_scalars(self._h.h, _lib.dptr(sq),
                                                           _lib.dptr(rho), _lib.dptr(xn)))
            self._cache["scalars"] = (float(sq[0]), float(rho[0]), float(xn[0]))
        return self._cache["scalars"]

    @property
    def sq_norm(self) -> float:
        return self._scalars()[0]

    def tracked_sq_norm(self) -> float:
        """Incrementally maintained squared Frobenius norm of the matrix."""
        return self._scalars()[0]

    @property
    def last_residual(self) -> float:
        return self._scalars()[1]

    @property
    def last_input_norm(self) -> float:
        return self._scalars()[2]

    @property
    def rank(self) -> int:
        """Current factor width (no transfer)."""
        return self._shape_all()[3]

    @property
    def singular_values(self) -> np.ndarray:
        """The installed singular values alone: r doubles, no basis download
        and no materialisation of the deferred bases (the per-tick metrics,
        metrics.py:86-93 / 122-145, need only these and the rank)."""
        if "factors" in self._cache:
            return self._cache["factors"].s
        if "s" not in self._cache:
            r = self._shape_all()[3]
            s = np.empty(r)
            _lib.check(self._h.lib.isvd_engine_get_factors(self._h.h, 0, None, _lib.dptr(s), None))
            self._cache["s"] = s
        return self._cache["s"]

    @property
    def factors(self) -> SvdFactors:
        if "factors" not in self._cache:
            _, m, n, r, _, _ = self._shape_all()
            u, s, v = np.empty((m, r)), np.empty(r), np.empty((n, r))
            _lib.check(self._h.lib.isvd_engine_get_factors(self._h.h, 0, _lib.dptr(u),
                                                           _lib.dptr(s), _lib.dptr(v)))
            self._cache["factors"] = SvdFactors(u, s, np.ascontiguousarray(v.T))
        return self._cache["factors"]

    @factors.setter
    def factors(self, f: SvdFactors) -> None:
        u = as_matrix(f.u, "u")
        s = as_vector(f.s, name="s")
        v = np.ascontiguousarray(as_matrix(f.vt, "vt").T)
        _lib.check(self._h.lib.isvd_engine_set_factors(self._h.h, 0, int(s.shape[0]),
                                                       _lib.dptr(u), _lib.dptr(s), _lib.dptr(v)))
        self._touch()

    @property
    def ref_subspace(self):
        if "ref" not in self._cache:
            has, rm, rr = C.c_int(), C.c_int(), C.c_int()
            _lib.check(self._h.lib.isvd_engine_has_reference(self._h.h, C.byref(has), C.byref(rm),
                                                             C.byref(rr)))
            ref = None
            if has.value:
                ref = np.empty((rm.value, rr.value))
                _lib.check(self._h.lib.isvd_engine_get_reference(self._h.h, 0, _lib.dptr(ref)))
            self._cache["ref"] = ref
        return self._cache["ref"]

    @ref_subspace.setter
    def ref_subspace(self, q) -> None:
        if q is None:
            _lib.check(self._h.lib.isvd_engine_put_reference(self._h.h, 0, 0, 0, None))
        else:
            q = as_matrix(q, "reference basis")
            _lib.check(self._h.lib.isvd_engine_put_reference(self._h.h, 0, q.shape[0], q.shape[1],
                                                             _lib.dptr(q)))
        self._touch()

    # ------------------------------------------------------------ events
    def row_append(self, x) -> None:
        """Append one row; exact up to truncation back to the work rank."""
        _, m, n, *_ = self._shape_all()
        x = as_vector(x, length=n, name="appended row")
        _lib.check(self._h.lib.isvd_engine_row_append(self._h.h, x.ctypes.data, 0))
        self._touch()

    def col_append(self, y) -> None:
        """Append one column (a row append of the transposed problem)."""
        _, m, n, *_ = self._shape_all()
        y = as_vector(y, length=m, name="appended column")
        _lib.check(self._h.lib.isvd_engine_col_append(self._h.h, y.ctypes.data, 0))
        self._touch()

    def rank_one_update(self, i: int, j: int, delta: float) -> None:
        """Add ``delta`` to entry (i, j) (projection semantics for the factors)."""
        _, m, n, *_ = self._shape_all()
        if not (0 <= i < m and 0 <= j < n):
            raise ValueError(f"index ({i}, {j}) out of bounds for shape ({m}, {n})")
        delta = float(delta)
        if not np.isfinite(delta):
            raise ValueError("delta must be finite")
        ii = np.array([int(i)], dtype=np.int64)
        jj = np.array([int(j)], dtype=np.int64)
        dd = np.array([delta])
        _lib.check(self._h.lib.isvd_engine_rank_one(self._h.h, ii.ctypes.data, jj.ctypes.data,
                                                    dd.ctypes.data, 0))
        self._touch()

    # ------------------------------------------------------- maintenance
    def refresh(self, store_reference: bool = False) -> None:
        """Recompute the truncated SVD of the tracked matrix (drift reset)."""
        _lib.check(self._h.lib.isvd_engine_refresh(self._h.h, int(bool(store_reference))))
        self._touch()

    def set_reference(self) -> None:
        """Store the current left basis as the drift reference."""
        _lib.check(self._h.lib.isvd_engine_set_reference(self._h.h))
        self._touch()

    def set_rank(self, k_new: int) -> None:
        """Change the work rank (decreases truncate now, increases apply at
        the next append or refresh)."""
        if k_new < 1:
            raise ValueError(f"work rank must be >= 1, got {k_new}")
        _lib.check(self._h.lib.isvd_engine_set_rank(self._h.h, int(k_new)))
        self._touch()

    # ------------------------------------------------- device-side metrics
    def _frob_error(self) -> float:
        out = np.empty(1)
        _lib.check(self._h.lib.isvd_engine_frob_error(self._h.h, _lib.dptr(out)))
        return float(out[0])

    def _angle(self, which: int, q=None) -> float | None:
        out = np.empty(1)
        if which == 0:
            _lib.check(self._h.lib.isvd_engine_angle(self._h.h, 0, None, 0, 0, _lib.dptr(out)))
            return None if out[0] < 0 else float(out[0])
        q = as_matrix(q, "basis")
        _lib.check(self._h.lib.isvd_engine_angle(self._h.h, 1, q.ctypes.data, int(q.shape[1]), 0,
                                                 _lib.dptr(out)))
        return float(out[0])

    def _oracle(self, w_keep: int):
        _, m, n, *_ = self._shape_all()
        nc = min(m, n)
        w = max(0, min(int(w_keep), nc))
        s = np.empty(nc)
        u = np.empty((m, w))
        _lib.check(self._h.lib.isvd_engine_oracle(self._h.h, w, _lib.dptr(s), _lib.dptr(u)))
        return s, u

    def set_lazy(self, on: bool) -> None:
        """Deferred left-basis rotation on (default) or off (eager per event)."""
        _lib.check(self._h.lib.isvd_engine_set_lazy(self._h.h, int(bool(on))))

    def set_vdefer(self, mode: int) -> None:
        """Deferred right-basis rotation on rank-1 updates: 0 off, 1 auto
        (batches >= 64 streams, the default), 2 whenever supported."""
        _lib.check(self._h.lib.isvd_engine_set_vdefer(self._h.h, int(mode)))

    @property
    def reortho_threshold(self) -> float:
        """Defect above which the guard re-factors (engine.py:30)."""
        return getattr(self, "_reortho_threshold", REORTHO_THRESHOLD)

    @reortho_threshold.setter
    def reortho_threshold(self, value: float) -> None:
        _lib.check(self._h.lib.isvd_engine_set_reortho_threshold(self._h.h, float(value)))
        self._reortho_threshold = float(value)

    def ortho_defects(self) -> tuple[float, float]:
        du, dv = np.empty(1), np.empty(1)
        _lib.check(self._h.lib.isvd_engine_ortho_defect(self._h.h, _lib.dptr(du), _lib.dptr(dv)))
        return float(du[0]), float(dv[0])

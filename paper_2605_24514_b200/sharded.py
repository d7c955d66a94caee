"""Row-sharded incremental SVD of one tall stream (BASELINE config 5b).

SURVEY.md 8(e) / north star: "for very tall matrices U is row-sharded, with
an NCCL-over-NVLink allreduce of the k-length projection vectors and k x k
Gram blocks".  Each rank of a ``torch.distributed`` process group holds a
contiguous block of rows of U and of the tracked matrix; s, V and the
deferred-window basis W are replicated and updated identically (same kernels
on the same inputs), so a row append needs no communication at all.  The
cross-rank sums libisvd asks for (isvd_engine_set_shard in include/isvd.h)
go through ``torch.distributed.all_reduce`` on the engine's CUDA stream:

  init / refresh   A^T A (n x n), two CholeskyQR Grams (k x k), ||A||^2
  column append    U^T y and ||y||^2 (k + 1), then ||z||^2
  rank-1 update    U[i, :] and A[i, j] from the owning rank (k + 1)
  metrics, signs   U Grams (k x k), ||A - U S V^T||^2, column-max packets

The last rank owns (stores) every appended row, so global row indices stay
contiguous per rank.  Observation calls are collective: every rank must make
them in the same order.  NCCL reduces device buffers in place; other backends
(gloo, for tests) stage through host memory.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .engine import _DeviceInputs, _Handle, _event_array, _is_device
from .linalg import SvdFactors


def shard_rows(m: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous block [row0, row0 + rows) of m rows for `rank` of `world`
    (sizes differ by at most one, larger blocks first)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank / world")
    base, extra = divmod(m, world)
    row0 = rank * base + min(rank, extra)
    return row0, base + (1 if rank < extra else 0)


class _DeviceBuffer:
    """Zero-copy view of a libisvd device buffer for torch.as_tensor."""

    def __init__(self, ptr: int, count: int):
        self.__cuda_array_interface__ = {"shape": (int(count),), "typestr": "<f8",
                                         "data": (int(ptr), False), "version": 3}


def make_allreduce(group=None):
    """The isvd_allreduce_fn callback over a torch.distributed group."""
    import torch
    import torch.distributed as dist

    backend = dist.get_backend(group)
    state = {"error": None}

    def _cb(ctx, buf, count, stream):
        try:
            t = torch.as_tensor(_DeviceBuffer(buf, count), device="cuda")
            with torch.cuda.stream(torch.cuda.ExternalStream(int(stream or 0))):
                if backend == "nccl":
                    dist.all_reduce(t, group=group)
                else:
                    h = t.cpu()
                    dist.all_reduce(h, group=group)
                    t.copy_(h)
            return 0
        except Exception as exc:  # reported through isvd_last_error as a failed call
            state["error"] = exc
            return 1

    return _lib.ALLREDUCE_FN(_cb), state


class ShardedSvdEngine:
    """One tall stream, rows sharded over the ranks of `group`.

    ``a_local`` is this rank's block of the initial matrix (rows
    [row0, row0 + m_local) of the global m_global x n matrix), a numpy array
    or a CUDA tensor.  Events take global arguments (a full row, a full
    column, global (i, j)); properties return this rank's rows of U."""

    def __init__(self, a_local, k: int, *, m_global: int, row0: int, group=None,
                 tol: float = 1e-10, rows_cap: int = 0, k_cap: int = 0, stream=None):
        import torch.distributed as dist

        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        on_dev = _is_device(a_local)
        if on_dev:
            src = a_local.contiguous()
            m_loc, n = (int(v) for v in src.shape)
        else:
            src = np.ascontiguousarray(np.asarray(a_local, dtype=np.float64))
            m_loc, n = src.shape
        if k < 1:
            raise ValueError(f"work rank must be >= 1, got {k}")
        self.owner = self.rank == self.world - 1
        cap = rows_cap if (rows_cap and self.owner) else 0
        self._h = _Handle(1, m_loc, n, k, tol, False, cap, 0, k_cap, stream)
        self._cb, self._cb_state = make_allreduce(group)
        _lib.check(self._h.lib.isvd_engine_set_shard(self._h.h, self.rank, self.world, int(row0),
                                                     int(m_global), int(self.owner),
                                                     C.cast(self._cb, C.c_void_p), None))
        self.row0 = int(row0)
        self.tol = float(tol)
        self._dev = _DeviceInputs(self._h)
        if on_dev:
            src = self._dev.check(src, "float64", (m_loc, n), "a_local")
            self._dev.before()
        self._check(self._h.lib.isvd_engine_init(self._h.h, _lib.vptr(src), int(on_dev)))

    def _check(self, rc):
        if rc != 0 and self._cb_state["error"] is not None:
            err, self._cb_state["error"] = self._cb_state["error"], None
            raise RuntimeError(f"allreduce failed: {err}") from err
        _lib.check(rc)

    # ------------------------------------------------------------ state
    def _info(self):
        r0, ml, mg = C.c_int64(), C.c_int(), C.c_int()
        _lib.check(self._h.lib.isvd_engine_shard_info(self._h.h, C.byref(r0), C.byref(ml),
                                                      C.byref(mg)))
        return r0.value, ml.value, mg.value

    @property
    def shape(self) -> tuple[int, int]:
        _, m, n, *_ = self._h.shape()
        return m, n

    @property
    def local_rows(self) -> int:
        return self._info()[1]

    @property
    def work_rank(self) -> int:
        return self._h.shape()[4]

    @property
    def step(self) -> int:
        return self._h.shape()[5]

    @property
    def cuda_stream(self) -> int:
        return self._h.stream()

    def scalars(self):
        sq, rho, xn = np.empty(1), np.empty(1), np.empty(1)
        _lib.check(self._h.lib.isvd_engine_get_scalars(self._h.h, _lib.dptr(sq), _lib.dptr(rho),
                                                       _lib.dptr(xn)))
        return float(sq[0]), float(rho[0]), float(xn[0])

    def scalars_async(self, out, slot: int = 0) -> None:
        _lib.check(self._h.lib.isvd_engine_scalars_async(self._h.h, _lib.vptr(out), int(slot)))

    def scalars_wait(self, slot: int = 0) -> None:
        _lib.check(self._h.lib.isvd_engine_scalars_wait(self._h.h, int(slot)))

    @property
    def sq_norm(self) -> float:
        return self.scalars()[0]

    @property
    def factors(self) -> SvdFactors:
        """(local rows of U, s, Vt) -- collective (sign canonicalisation)."""
        _, ml, _ = self._info()
        r = self._h.shape()[3]
        n = self.shape[1]
        u, s, v = np.empty((ml, r)), np.empty(r), np.empty((n, r))
        self._check(self._h.lib.isvd_engine_get_factors(self._h.h, 0, _lib.dptr(u), _lib.dptr(s),
                                                        _lib.dptr(v)))
        return SvdFactors(u, s, np.ascontiguousarray(v.T))

    def gather_factors(self) -> SvdFactors:
        """The whole U on every rank (all_gather of the row blocks)."""
        import torch
        import torch.distributed as dist

        f = self.factors
        sizes = [None] * self.world
        dist.all_gather_object(sizes, f.u.shape[0], group=self.group)
        mx = max(sizes)
        buf = torch.zeros((mx, f.u.shape[1]), dtype=torch.float64)
        buf[:f.u.shape[0]] = torch.from_numpy(f.u)
        dev = "cuda" if dist.get_backend(self.group) == "nccl" else "cpu"
        buf = buf.to(dev)
        outs = [torch.empty_like(buf) for _ in range(self.world)]
        dist.all_gather(outs, buf, group=self.group)
        u = np.concatenate([o.cpu().numpy()[:sz] for o, sz in zip(outs, sizes)], axis=0)
        return SvdFactors(u, f.s, f.vt)

    def synchronize(self) -> None:
        _lib.check(self._h.lib.isvd_engine_synchronize(self._h.h))

    def flush(self) -> None:
        self._check(self._h.lib.isvd_engine_flush(self._h.h))

    def snapshot(self) -> None:
        _lib.check(self._h.lib.isvd_engine_snapshot(self._h.h))

    def restore(self) -> None:
        _lib.check(self._h.lib.isvd_engine_restore(self._h.h))

    # ------------------------------------------------------------ events
    def row_append(self, x) -> None:
        n = self.shape[1]
        if _is_device(x):
            src = self._dev.check(x.reshape(1, -1), "float64", (1, n), "appended row")
            self._dev.before()
            self._check(self._h.lib.isvd_engine_row_append(self._h.h, _lib.vptr(src), 1))
            self._dev.after(src)
            return
        x = np.asarray(x, dtype=np.float64).reshape(1, -1)
        src, _ = _event_array(x, (1, n), "appended row")
        self._check(self._h.lib.isvd_engine_row_append(self._h.h, _lib.vptr(src), 0))

    def col_append(self, y) -> None:
        """y: the full global column (length m_global); this rank uses its rows."""
        m = self.shape[0]
        r0, ml, _ = self._info()
        if _is_device(y):
            if tuple(y.shape) not in ((m,), (1, m)):
                raise ValueError(f"appended column has shape {tuple(y.shape)}, expected ({m},)")
            part = self._dev.check(y.reshape(-1)[r0:r0 + ml].reshape(1, ml), "float64", (1, ml),
                                   "appended column")
            self._dev.before()
            self._check(self._h.lib.isvd_engine_col_append(self._h.h, _lib.vptr(part), 1))
            self._dev.after(part)
            return
        else:
            arr = np.asarray(y, dtype=np.float64).reshape(-1)
            if arr.shape != (m,):
                raise ValueError(f"appended column has shape {arr.shape}, expected ({m},)")
            part = np.ascontiguousarray(arr[r0:r0 + ml]).reshape(1, ml)
        src, _ = _event_array(part, (1, ml), "appended column")
        self._check(self._h.lib.isvd_engine_col_append(self._h.h, _lib.vptr(src), 0))

    def rank_one_update(self, i: int, j: int, delta: float) -> None:
        ii = np.array([int(i)], dtype=np.int64)
        jj = np.array([int(j)], dtype=np.int64)
        dd = np.array([float(delta)], dtype=np.float64)
        self._check(self._h.lib.isvd_engine_rank_one(self._h.h, _lib.vptr(ii), _lib.vptr(jj),
                                                     _lib.vptr(dd), 0))

    def refresh(self, store_reference: bool = False) -> None:
        self._check(self._h.lib.isvd_engine_refresh(self._h.h, int(bool(store_reference))))

    def set_reference(self) -> None:
        self._check(self._h.lib.isvd_engine_set_reference(self._h.h))

    # ------------------------------------------------------------ metrics
    def frob_error(self) -> float:
        out = np.empty(1)
        self._check(self._h.lib.isvd_engine_frob_error(self._h.h, _lib.dptr(out)))
        return float(out[0])

    def ortho_defect(self) -> tuple[float, float]:
        du, dv = np.empty(1), np.empty(1)
        self._check(self._h.lib.isvd_engine_ortho_defect(self._h.h, _lib.dptr(du), _lib.dptr(dv)))
        return float(du[0]), float(dv[0])

    def angle_to_reference(self) -> float | None:
        out = np.empty(1)
        self._check(self._h.lib.isvd_engine_angle(self._h.h, 0, None, 0, 0, _lib.dptr(out)))
        return None if out[0] < 0 else float(out[0])

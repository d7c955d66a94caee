"""Tall-matrix path on the GPU: the DMMA Gram / GEMM contractions, the
Gram-based thin SVD (init / refresh / oracle of BASELINE configs 4 and 5b)
and the k = 128 engine on a reduced-height config 5b ("pin
parity at reduced m, same code path")."""

import numpy as np
import pytest
import torch

from conftest import rel_err, sine_angle
from oracle import OracleEngine as OEngine
from oracle import full_svd as o_full_svd
from paper_2605_24514_b200 import BatchedSvdEngine, SvdEngine, _lib, full_svd, truncated_svd
from paper_2605_24514_b200.linalg import _device_svd, orthonormality_defect

pytestmark = pytest.mark.gpu

DEV = torch.device("cuda", 0)


def _lib_handle():
    return _lib.load()


@pytest.mark.parametrize("rows, wa, wb, same", [
    (1, 1, 1, True), (7, 3, 5, False), (100, 33, 70, False), (513, 64, 64, True),
    (5000, 128, 128, True), (70001, 200, 64, False), (3, 130, 5, False), (40000, 129, 129, True),
])
def test_gram_matches_fp64(rows, wa, wb, same):
    g = torch.Generator(device="cpu").manual_seed(rows + wa * 7 + wb)
    xa = torch.randn(rows, wa + 3, dtype=torch.float64, generator=g).to(DEV)
    xb = xa if same else torch.randn(rows, wb + 1, dtype=torch.float64, generator=g).to(DEV)
    wb_eff = wa if same else wb
    out = torch.empty(wa, wb_eff, dtype=torch.float64, device=DEV)
    lib = _lib_handle()
    _lib.check(lib.isvd_gram(rows, wa, wb_eff, xa.data_ptr(), xa.shape[1], xb.data_ptr(),
                             xb.shape[1], out.data_ptr(), None))
    torch.cuda.synchronize()
    ref = xa[:, :wa].cpu().numpy().T @ xb[:, :wb_eff].cpu().numpy()
    scale = np.sqrt(rows) * 1e-14 * max(1.0, np.abs(ref).max())
    np.testing.assert_allclose(out.cpu().numpy(), ref, rtol=0, atol=scale * 10)
    if same:
        o = out.cpu().numpy()
        assert np.array_equal(o, o.T)  # mirrored, bit-symmetric


@pytest.mark.parametrize("rows, n, wc", [(1, 1, 1), (65, 33, 17), (1000, 1024, 128),
                                         (300, 5, 200), (20001, 96, 64)])
def test_gemm_tall_matches_fp64(rows, n, wc):
    g = torch.Generator(device="cpu").manual_seed(rows * 3 + n + wc)
    x = torch.randn(rows, n + 2, dtype=torch.float64, generator=g).to(DEV)
    q = torch.randn(n, wc + 5, dtype=torch.float64, generator=g).to(DEV)
    c = torch.full((rows, wc + 1), 7.0, dtype=torch.float64, device=DEV)
    lib = _lib_handle()
    _lib.check(lib.isvd_gemm_tall(rows, n, wc, x.data_ptr(), x.shape[1], q.data_ptr(), q.shape[1],
                                  c.data_ptr(), c.shape[1], None))
    torch.cuda.synchronize()
    ref = x[:, :n].cpu().numpy() @ q[:, :wc].cpu().numpy()
    got = c.cpu().numpy()
    np.testing.assert_allclose(got[:, :wc], ref, rtol=0, atol=1e-13 * np.sqrt(n) * 10)
    assert np.all(got[:, wc] == 7.0)  # pitch respected


def _tall_matrix(m, n, rank, noise, seed, decay=None):
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((m, rank))
    y = rng.standard_normal((n, rank))
    if decay is not None:
        x = x * decay ** np.arange(rank)
    return x @ y.T + noise * rng.standard_normal((m, n))


@pytest.mark.parametrize("m, n, rank, k", [(16384, 1024, 64, 64), (20000, 512, 40, 128)])
def test_gram_path_svd_matches_lapack(m, n, rank, k):
    a = _tall_matrix(m, n, rank, 1e-2, seed=m + n)
    f = truncated_svd(a, k)
    fo = o_full_svd(a)
    w = min(k, n)
    assert rel_err(f.s[:rank], fo.s[:rank]) < 1e-9
    assert sine_angle(f.u[:, :rank], fo.u[:, :rank]) < 1e-6
    assert sine_angle(f.vt[:rank].T, fo.vt[:rank].T) < 1e-6
    # noise directions are clustered; their singular values still match
    assert rel_err(f.s[:w], fo.s[:w]) < 1e-9
    assert orthonormality_defect(f.u) <= 1e-10
    assert orthonormality_defect(f.vt.T) <= 1e-10
    lead = np.argmax(np.abs(f.u), axis=0)
    assert np.all(f.u[lead, np.arange(w)] >= 0.0)
    # full spectrum (the oracle's E_opt input): head from the Ritz step, tail
    # from the Gram eigenvalues
    _, s_all, _ = _device_svd(a, k)
    assert rel_err(s_all, fo.s) < 1e-7
    e_opt = np.linalg.norm(s_all[k:]) if k < n else 0.0
    assert abs(e_opt - np.linalg.norm(fo.s[k:])) <= 1e-9 * max(1.0, np.linalg.norm(fo.s))
    # all n triplets (w > kGramMaxW) take the blocked-Jacobi path
    g = full_svd(a)
    assert rel_err(g.s, fo.s) < 1e-10


def test_gram_path_rank_deficient():
    a = _tall_matrix(16384, 1024, 20, 0.0, seed=5)
    f = truncated_svd(a, 32)
    fo = o_full_svd(a)
    assert rel_err(f.s[:20], fo.s[:20]) < 1e-9
    assert np.all(f.s[20:] == 0.0)
    assert orthonormality_defect(f.u) <= 1e-10  # dead columns completed
    assert sine_angle(f.u[:, :20], fo.u[:, :20]) < 1e-6


def test_cfg5b_reduced_matches_oracle():
    """Config 5b at m = 2^15: rank-128 + small noise, k = 128, row appends
    l.Y^T; same code path as the full size (Gram init, k = 128
    secular core, deferred U, DMMA rotation)."""
    m, n, k = 1 << 15, 1024, 128
    rng = np.random.default_rng([0, 55])
    x = rng.standard_normal((m, k))
    y = rng.standard_normal((n, k))
    a0 = x @ y.T + 1e-3 * rng.standard_normal((m, n))
    rows = rng.standard_normal((24, k)) @ y.T
    eng = SvdEngine(a0, k, capacity=(m + 32, n, k))
    ora = OEngine(a0, k)
    assert rel_err(eng.factors.s, ora.factors.s) < 1e-9
    for t in range(rows.shape[0]):
        eng.row_append(rows[t])
        ora.row_append(rows[t])
    f, fo = eng.factors, ora.factors
    assert f.u.shape == fo.u.shape == (m + 24, k)
    assert rel_err(f.s, fo.s) < 1e-9
    assert sine_angle(f.u, fo.u) < 1e-6
    assert sine_angle(f.vt.T, fo.vt.T) < 1e-6
    assert orthonormality_defect(f.u) <= 1e-9
    assert abs(eng.sq_norm - ora.sq_norm) <= 1e-12 * ora.sq_norm
    assert abs(eng.last_residual - ora.last_residual) <= 1e-6 * max(1.0, ora.last_input_norm)


def test_cfg5b_full_size_invariants():
    """Full 4,194,304 x 1024 (k = 128, 256 row appends, device-resident inputs):
    orthonormality <= 1e-8, the N_t identity and exact reconstruction of the
    appended rows' span (rows l.Y^T lie in the kept right subspace)."""
    m, n, k, T = 1 << 22, 1024, 128, 256
    g = torch.Generator(device=DEV).manual_seed(5)
    y = torch.randn(n, k, dtype=torch.float64, device=DEV, generator=g)
    a0 = torch.empty(m, n, dtype=torch.float64, device=DEV)
    step = 1 << 18
    for c in range(0, m, step):  # chunked: keeps the generator's temporaries small
        x = torch.randn(step, k, dtype=torch.float64, device=DEV, generator=g)
        a0[c:c + step] = x @ y.T + 1e-3 * torch.randn(step, n, dtype=torch.float64, device=DEV,
                                                     generator=g)
    n0 = float(torch.linalg.vector_norm(a0) ** 2)
    rows = torch.randn(T, k, dtype=torch.float64, device=DEV, generator=g) @ y.T
    eng = BatchedSvdEngine(a0.view(1, m, n), k, m_cap=m + T + 1, k_cap=k)
    del a0
    torch.cuda.empty_cache()
    for t in range(T):
        eng.row_append(rows[t:t + 1])
    eng.flush()
    eng.synchronize()
    assert eng.shape == (m + T, n)
    n_expect = n0 + float((rows * rows).sum())
    sq, rho, xn = eng.scalars()
    assert abs(float(sq[0]) - n_expect) <= 1e-11 * n_expect
    du, dv = eng.ortho_defect()
    assert float(du[0]) <= 1e-8 and float(dv[0]) <= 1e-8
    # the last appended row l.Y^T lies in span(Y); V is tilted from it only by
    # the 1e-3 noise (~noise / sigma_k ~ 3e-5)
    assert float(rho[0]) <= 1e-3 * float(xn[0])

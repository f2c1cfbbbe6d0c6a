"""Pins for the oracle on graded layer-adapted meshes: the Bakhvalov-Shishkin
mesh (reading R21), the 5-point stencil with coordinate-difference widths, geometric
bilinear interpolation on graded corner levels ("interpolation that accounts for the
mesh spacing"), and the method on such meshes (Remark rem:not just S-meshes: the
theory "covers ... graded (e.g., Bakhvalov) meshes").  Expected values come from closed forms,
numpy brute force and mathematical invariants, never from the oracle or the CUDA path."""
import numpy as np
import pytest

import oracle
import spp_inputs as si

from test_oracle_2d import _dense, _dense_level, _mhat, _region


def _bs(name, N, eps, sigma=2.0, bx=1.0, by=1.0, **kw):
    cfg = si.config(name, N=N, eps=eps)
    x = oracle.mesh_bs(N, cfg.eps, sigma, bx)
    y = oracle.mesh_bs(N, cfg.eps, sigma, by)
    c1, c2, r, f = si.sample_2d(cfg, x, y)
    return cfg, x, y, (c1, c2, r, f), oracle.Oracle2D(N, cfg.eps, x, y, c1, c2, r, **kw)


@pytest.mark.parametrize("N,eps,sigma,beta", [(16, 1e-3, 2.0, 1.0), (256, 1e-8, 2.0, 1.0), (1024, 1e-6, 2.5, 1.99),
                                              (64, 1e-2, 2.0, 1.0)])
def test_bs_mesh_properties(N, eps, sigma, beta):
    """Graded on [0, tau] with tau = sigma eps ln(N) / beta at index N/2 (the transition point of
    eq:tau exponential, which the block structure needs), uniform on
    [tau, 1]; the layer widths grow from ~(2 sigma eps/beta)/N to ~sigma eps/beta (mesh-generating
    function -ln(1 - 2(1-1/N) t): derivative ratio N between t = 0 and t = 1/2)."""
    x = oracle.mesh_bs(N, eps, sigma, beta)
    n = N // 2
    tau = sigma * eps * np.log(N) / beta
    h = np.diff(x)
    assert x[0] == 0.0 and x[N] == 1.0 and np.all(h > 0)
    if tau > 0.5:
        assert np.allclose(x, np.arange(N + 1) / N, rtol=0, atol=1e-15)
        return
    assert np.isclose(x[n], tau, rtol=1e-15)
    assert np.allclose(h[n:], (1 - tau) / n, rtol=1e-12)
    assert np.all(np.diff(h[:n]) > 0)                                  # graded: widths increase
    s = sigma * eps / beta
    assert np.isclose(h[0], 2 * s / N, rtol=2.0 / N)                   # phi'(0) / N
    assert N / 4 <= h[n - 1] / h[0] <= N                               # phi'(1/2) / phi'(0) ~ N
    # the same transition point as the Shishkin mesh: the regions C, X, Y, I coincide
    assert x[n] == oracle.mesh(N, eps, sigma, beta)[n]


def _stencil_dense(x, y, eps, c1, c2, r):
    """The upwind 5-point stencil of P:972-981 on an arbitrary tensor mesh, h_i = x_i - x_{i-1},
    hbar_i = (h_i + h_{i+1})/2 (written out here in numpy, independently of the oracle)."""
    N = len(x) - 1
    m = N - 1
    A = np.zeros((m * m, m * m))
    for j in range(1, N):
        for i in range(1, N):
            hi, hi1 = x[i] - x[i - 1], x[i + 1] - x[i]
            kj, kj1 = y[j] - y[j - 1], y[j + 1] - y[j]
            hb, kb = (hi + hi1) / 2, (kj + kj1) / 2
            p = (j - 1) * m + (i - 1)
            a1, a2 = c1[j - 1, i - 1], c2[j - 1, i - 1]
            A[p, p] = eps / hb * (1 / hi + 1 / hi1) + eps / kb * (1 / kj + 1 / kj1) + a1 / hi1 + a2 / kj1 + r[j - 1, i - 1]
            if i > 1:
                A[p, p - 1] = -eps / (hb * hi)
            if i < m:
                A[p, p + 1] = -eps / (hb * hi1) - a1 / hi1
            if j > 1:
                A[p, p - m] = -eps / (kb * kj)
            if j < m:
                A[p, p + m] = -eps / (kb * kj1) - a2 / kj1
    return A


@pytest.mark.parametrize("eps", [1e-2, 1e-6])
def test_bs_operator_brute_force(eps):
    N = 16
    cfg, x, y, (c1, c2, r, f), P = _bs("cfg4", N, eps)
    A = _dense(P)
    B = _stencil_dense(x, y, eps, c1, c2, r)
    assert np.allclose(A, B, rtol=1e-12, atol=1e-12 * np.abs(B).max())
    d = np.diag(A)
    off = A - np.diag(d)
    assert np.all(d > 0) and np.all(off <= 0) and np.all(np.abs(off).sum(1) <= d)
    ue = np.linalg.solve(B, f.ravel())
    assert np.linalg.norm(P.direct(f).ravel() - ue) <= 1e-11 * np.linalg.norm(ue)


def test_bs_interpolation_is_geometric():
    """On a graded corner the prolongation is the linear interpolant in the level's coordinates:
    it reproduces g = x y (zero on the Dirichlet sides x = 0, y = 0) exactly, which weights of 1/2
    would not; the restriction is S_c^{-1} P^T S_f (adjointness)."""
    N = 64
    cfg, x, y, ins, P = _bs("cfg5", N, 1e-6, bx=1.0, by=2.0)
    n = N // 2
    f0, c1_ = P.level_coef(0), P.level_coef(1)
    nf, nc = f0["n"], c1_["n"]
    xf, yf = x[1:n + 1], y[1:n + 1]                                   # level 0 nodes
    xc, yc = x[2:n + 1:2], y[2:n + 1:2]                               # level 1 nodes
    gf = np.outer(yf, xf)
    gc = np.outer(yc, xc)
    Pg = P.prolong_add(0, gc, np.zeros((nf, nf)))
    assert np.allclose(Pg, gf, rtol=1e-13, atol=0)
    uniform = 0.5 * (gc[:, :-1] + gc[:, 1:])                          # what weights 1/2 would give
    assert not np.allclose(uniform[-1], gf[-1, 2:nf - 1:2], rtol=1e-6, atol=0)
    Sf = np.outer(f0["kb"][1:nf + 1], f0["hb"][1:nf + 1])
    Sc = np.outer(c1_["kb"][1:nc + 1], c1_["hb"][1:nc + 1])
    v = si.random_field(61, (nf, nf))
    ec = si.random_field(62, (nc, nc))
    Pe = P.prolong_add(0, ec, np.zeros((nf, nf)))
    assert np.isclose(np.sum(Pe * Sf * v), np.sum(ec * Sc * P.restrict(0, v)), rtol=1e-13)


def test_bs_block_preconditioner_and_corner_solve():
    """eq:2D blocks on a graded mesh: with the corner solved to rounding, M^{-1} q
    is a dense solve with M-hat; the corner multigrid converges to A_CC^{-1} b."""
    N = 16
    cfg, x, y, (c1, c2, r, f), P = _bs("cfg4", N, 1e-8, mg_fixed=300)   # corner solved to rounding
    A = _dense(P)
    M = _mhat(A, N)
    q = si.random_field(63, (N - 1, N - 1))
    z = P.precond(q).ravel()
    # the graded mesh makes M-hat ill-conditioned (widths 1e-11 .. 1e-1, cond ~ 3e9), so the check
    # is the scaled backward error of z as a solution of M-hat z = q, not a forward comparison
    Dm = np.abs(np.diag(M))
    assert np.linalg.norm((M @ z - q.ravel()) / Dm) <= 1e-13 * np.linalg.norm(q.ravel() / Dm)
    n = N // 2
    b = si.random_field(64, (n, n))
    zc, cyc, cap = P.corner_solve(b)
    reg = np.array([_region(i, j, n) for j in range(1, N) for i in range(1, N)])
    AC = A[np.ix_(reg == 0, reg == 0)]
    assert np.allclose(_dense_level(P, 0), AC, rtol=1e-13, atol=0)
    Dc = np.abs(np.diag(AC))
    assert not cap and np.linalg.norm((AC @ zc.ravel() - b.ravel()) / Dc) <= 1e-13 * np.linalg.norm(b.ravel() / Dc)


def test_bs_first_order_convergence_and_fgmres():
    """eq:exponential_MMS on Bakhvalov-Shishkin meshes: the upwind error decays at
    the full first order N^{-1} (error ratio -> 2 per doubling, faster than the N^{-1} ln N of the
    Shishkin mesh, whose ratios are 2 ln N / ln 2N < 1.9 here), and the paper-stopped FGMRES
    iterate has the discretization error of the exact discrete solution."""
    eps = 1e-6
    errs = []
    for N in (64, 128, 256):
        cfg, x, y, (c1, c2, r, f), P = _bs("exp2d", N, eps, sigma=2.5, bx=1.99, by=2.99)
        ue = si.exact_solution(cfg, x, y)
        ud = P.direct(f)
        errs.append(np.max(np.abs(ud - ue)))
        res = P.solve(f, weighted=0, stop_abs=1, tol=cfg.tol, maxit=200)
        assert res["converged"]
        assert abs(np.max(np.abs(res["u"] - ue)) - errs[-1]) <= 0.02 * errs[-1]
        P.close()
    ratios = [errs[k] / errs[k + 1] for k in range(2)]
    assert all(1.9 <= q <= 2.1 for q in ratios), ratios
    assert all(2 * np.log(N) / np.log(2 * N) < 1.9 for N in (64, 128))


@pytest.mark.parametrize("name,eps", [("cfg4", 1e-8), ("cfg5", 1e-4)])
def test_bs_fgmres_deep_check_vs_direct(name, eps):
    N = 64
    cfg, x, y, (c1, c2, r, f), P = _bs(name, N, eps)
    res = P.solve(f, weighted=1, tol=1e-12, maxit=300)
    ud = P.direct(f)
    assert res["converged"]
    assert np.linalg.norm(res["u"] - ud) <= 1e-9 * np.linalg.norm(ud)


def test_bs_iterations_eps_robust():
    """Remark rem:not just S-meshes: the bound of Theorem big_bound holds on graded
    meshes, so for eps N small the FGMRES counts do not grow as eps -> 0."""
    N = 128
    its = []
    for eps in (1e-6, 1e-8, 1e-10):
        cfg, x, y, (c1, c2, r, f), P = _bs("cfg4", N, eps)
        its.append(P.solve(f, weighted=1, tol=1e-8)["iters"])
        P.close()
    assert max(its) - min(its) <= 3 and max(its) <= 20, its

"""Pins for the oracle's parabolic-layer variant (c2 = 0): the paper's own
Tables 3 and 4 -- discretization errors to 4 digits and FGMRES counts exactly -- and
"3 V-cycles" per corner solve; the semi-coarsening Galerkin hierarchy against its
definitions, written out in numpy from the dense operator: the operator-induced interpolation of
the North-South collapsed stencil, R = P^T and A_c = R A P,
the FE row scaling of the finest grid, downstream point Gauss-Seidel."""
import numpy as np
import pytest

import oracle
import spp_inputs as si
from conftest import load_table, rounds_to

T3 = load_table("table3_par_errors.txt")
T4 = load_table("table4_par_iters.txt")


def _par(N, eps, **kw):
    cfg = si.config("par2d", N=N, eps=eps)
    x = oracle.mesh(N, cfg.eps, cfg.sigma, cfg.beta_x)          # eq:tau parabolic
    y = oracle.mesh(N, cfg.eps_y, cfg.sigma, cfg.beta_y)        # tau_y = sigma sqrt(eps) ln N
    c1, c2, r, f = si.sample_2d(cfg, x, y)
    kw.setdefault("mg_red", 1e-2)                               # "a relative factor of 10^2"
    return cfg, x, y, (c1, c2, r, f), oracle.Oracle2D(N, cfg.eps, x, y, c1, c2, r, **kw)


def test_parabolic_mesh_and_manufactured_solution():
    """tau_x = min(1/2, sigma eps ln N / C), tau_y = min(1/2, sigma sqrt(eps) ln N) with sigma = 5/2
    (eq:tau parabolic); u* vanishes on the boundary; the discrete operator with c2 = 0 keeps the
    M-matrix structure (c_{2,ij} >= 0)."""
    N, eps = 64, 1e-6
    cfg, x, y, (c1, c2, r, f), P = _par(N, eps)
    assert np.isclose(x[N // 2], 2.5 * eps * np.log(N) / 0.99, rtol=1e-14)
    assert np.isclose(y[N // 2], 2.5 * np.sqrt(eps) * np.log(N), rtol=1e-14)
    xx = np.array([0.0, 0.3, 1.0])
    u = si.exact_solution(si.config("par2d", N=4, eps=eps), xx, xx)            # interior node 0.3
    assert u.shape == (1, 1)
    edge = si.exact_solution(si.config("par2d", N=4, eps=eps), np.array([0, 1e-12, 1]), np.array([0, 0.5, 1]))
    assert abs(edge[0, 0]) < 1e-6                                # ~ 0 at the x = 0 boundary
    assert P.parabolic and np.all(c2 == 0)


@pytest.mark.parametrize("col,N", [(0, 128), (1, 256), (2, 512)])
def test_tables_3_4_parabolic(col, N):
    """FGMRES counts (exact) and max-norm errors (4 digits) for eq:parabolic_MMS with
    the paper's stop ||R||_2 <= 10 N^{-1} ln N; the corner reaches its 10^2 reduction in
    3 V-cycles.  12 of 12 cells."""
    for eps in sorted(T4):
        cfg, x, y, (c1, c2, r, f), P = _par(N, eps)
        res = P.solve(f, weighted=0, stop_abs=1, tol=cfg.tol, maxit=100)
        assert res["iters"] == int(T4[eps][col]), (N, eps, res["iters"])
        err = np.max(np.abs(res["u"] - si.exact_solution(cfg, x, y)))
        assert rounds_to(err, T3[eps][col]), (N, eps, err, T3[eps][col])
        assert set(res["cycle_log"]) == {3}, set(res["cycle_log"])
        P.close()


@pytest.mark.slow
@pytest.mark.parametrize("col,N", [(3, 1024), (4, 2048)])
def test_tables_3_4_parabolic_large(col, N):
    """The two largest columns.  Where every corner solve takes the paper's 3 cycles
    (6 of 8 cells) the count is exact and the error matches to 4 digits; in the other two cells
    (N = 1024, eps = 1e-5; N = 2048, eps = 1e-6 -- the top-right region of Table 4 where eps N is
    not small) the 10^2 reduction is met after 2 cycles in some applies and the count
    is one above the paper's (reading R22): the north_star bar of +-1."""
    for eps in sorted(T4):
        cfg, x, y, (c1, c2, r, f), P = _par(N, eps)
        res = P.solve(f, weighted=0, stop_abs=1, tol=cfg.tol, maxit=100)
        want = int(T4[eps][col])
        assert abs(res["iters"] - want) <= 1, (N, eps, res["iters"])
        if set(res["cycle_log"]) == {3}:
            assert res["iters"] == want, (N, eps, res["iters"])
            err = np.max(np.abs(res["u"] - si.exact_solution(cfg, x, y)))
            assert rounds_to(err, T3[eps][col]), (N, eps, err, T3[eps][col])
        P.close()


def _dense_plevel(P, l):
    """the level-l operator as a dense matrix, from its nine-point stencil"""
    a = P.plevel_stencil(l)
    ny, nx, _ = a.shape
    A = np.zeros((nx * ny, nx * ny))
    for j in range(ny):
        for i in range(nx):
            for dj in (-1, 0, 1):
                for di in (-1, 0, 1):
                    if 0 <= i + di < nx and 0 <= j + dj < ny:
                        A[j * nx + i, (j + dj) * nx + i + di] = a[j, i, (dj + 1) * 3 + di + 1]
                    else:
                        assert a[j, i, (dj + 1) * 3 + di + 1] == 0.0
    return A


def _interp_from_dense(A, nx, ny):
    """P of P:1231-1243 from a dense level operator: odd (1-based) i interpolates from the coarse
    nodes at i-1, i+1 with minus the W / E column sums over the centre column sum (North-South
    collapse); even i is the coarse node i/2."""
    nc = nx // 2
    Pm = np.zeros((nx * ny, nc * ny))
    for j in range(ny):
        for i in range(1, nx + 1):
            row = j * nx + (i - 1)
            if i % 2 == 0:
                Pm[row, j * nc + i // 2 - 1] = 1.0
                continue
            col = lambda ii: sum(A[row, jj * nx + ii - 1] for jj in (j - 1, j, j + 1) if 0 <= jj < ny and 1 <= ii <= nx)
            den = col(i)
            if (i - 1) // 2 >= 1:
                Pm[row, j * nc + (i - 1) // 2 - 1] = -col(i - 1) / den
            Pm[row, j * nc + (i + 1) // 2 - 1] = -col(i + 1) / den
    return Pm


def test_galerkin_hierarchy_matches_definitions():
    N, eps = 32, 1e-6
    cfg, x, y, ins, P = _par(N, eps)
    n = N // 2
    assert P.plevels == 3 and [P.plevel_shape(l) for l in range(3)] == [(16, 16), (16, 8), (16, 4)]
    # finest: A_CC with row (i,j) scaled by hbar_i kbar_j
    g, c0 = P.coef(), P.level_coef(0)
    A0 = _dense_plevel(P, 0)
    from test_oracle_2d import _dense, _region
    A = _dense(P)
    reg = np.array([_region(i, j, n) for j in range(1, N) for i in range(1, N)])
    S = np.outer(c0["kb"][1:n + 1], c0["hb"][1:n + 1]).ravel()
    assert np.allclose(A0, S[:, None] * A[np.ix_(reg == 0, reg == 0)], rtol=1e-14, atol=0)
    for l in range(P.plevels - 1):
        Al = _dense_plevel(P, l)
        ny, nx = P.plevel_shape(l)
        Pm = _interp_from_dense(Al, nx, ny)
        Ac = _dense_plevel(P, l + 1)
        assert np.allclose(Ac, Pm.T @ Al @ Pm, rtol=1e-12, atol=1e-12 * np.abs(Ac).max())
        ec = si.random_field(70 + l, (ny, nx // 2))
        assert np.allclose(P.pprolong_add(l, ec, np.zeros((ny, nx))).ravel(), Pm @ ec.ravel(), rtol=1e-14, atol=0)
        rv = si.random_field(80 + l, (ny, nx))
        assert np.allclose(P.prestrict(l, rv).ravel(), Pm.T @ rv.ravel(), rtol=1e-13, atol=1e-15)
    del g


@pytest.mark.parametrize("l", [0, 1])
def test_parabolic_gs_is_downstream_triangular_solve(l):
    """downstream point GS from the top-right to the bottom-left point: the new value
    uses E and the whole row above (NW, N, NE), the old W, SW, S, SE."""
    cfg, x, y, ins, P = _par(32, 1e-7)
    Al = _dense_plevel(P, l)
    ny, nx = P.plevel_shape(l)
    up = np.zeros_like(Al)
    for p in range(nx * ny):
        for q in np.nonzero(Al[p])[0]:
            if q >= p:                   # (j' > j) or (j' == j and i' >= i): already swept
                up[p, q] = Al[p, q]
    low = up - Al
    b = si.random_field(90 + l, (ny, nx)).ravel()
    e0 = si.random_field(95 + l, (ny, nx)).ravel()
    want = np.linalg.solve(up, b + low @ e0)
    assert np.allclose(P.pgs(l, b, e0).ravel(), want, rtol=1e-12, atol=1e-12 * np.abs(want).max())


def test_parabolic_corner_mg_converges_and_is_linear():
    N = 32
    cfg, x, y, ins, P = _par(N, 1e-6, mg_red=1e-14, mg_cap=300)
    n = N // 2
    b = si.random_field(99, (n, n))
    z, cyc, cap = P.corner_solve(b)
    from test_oracle_2d import _dense, _region
    A = _dense(P)
    reg = np.array([_region(i, j, n) for j in range(1, N) for i in range(1, N)])
    AC = A[np.ix_(reg == 0, reg == 0)]
    zz = np.linalg.solve(AC, b.ravel())
    assert not cap and np.linalg.norm(z.ravel() - zz) <= 1e-11 * np.linalg.norm(zz)
    v1, v10 = P.pvcycle(0, b), P.pvcycle(0, 10 * b)
    assert np.allclose(v10, 10 * v1, rtol=1e-13, atol=1e-13 * np.abs(v10).max())

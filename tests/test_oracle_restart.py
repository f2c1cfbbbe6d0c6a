"""Pins for the oracle's restarted FGMRES(m) (SURVEY 8(b) `restart`, reading R23).

The paper runs GMRES without restarts; FGMRES(m) is the library option for solves whose
Krylov basis would not fit in memory.  What fixes it is the definition of a GMRES(m)
cycle (Saad 2003, Alg. 6.9 restarted): from the current iterate x_c and its residual
r_c = W (f - A x_c), the next iterate is x_c + M^{-1} D Q t, where Q spans the Krylov space
K_m(B, r_c) of B = W A M^{-1} D and t minimises ||r_c - B Q t||_2.  With a fixed number of corner
cycles the preconditioner is a linear map, so every cycle can be written out with dense numpy
linear algebra (QR + least squares) on a small mesh and compared with the oracle's iterate.
The operator and the preconditioner themselves are pinned in test_oracle_2d.py."""
import numpy as np

import oracle
import spp_inputs as si


def _mk(name, N, eps, **kw):
    cfg = si.config(name, N=N, eps=eps)
    x = oracle.mesh(N, cfg.eps, 2.0, 1.0)
    c1, c2, r, f = si.sample_2d(cfg, x, x)
    P = oracle.Oracle2D(N, cfg.eps, x, x, c1, c2, r, **kw)
    return cfg, f, P


def _cols(op, n):
    M = np.zeros((n, n))
    for k in range(n):
        e = np.zeros(n)
        e[k] = 1.0
        M[:, k] = np.asarray(op(e)).ravel()
    return M


def test_restart_at_or_above_the_count_is_the_unrestarted_solve():
    cfg, f, P = _mk("cfg4", 32, 1e-8)
    a = P.solve(f, tol=1e-10)
    for m in (a["iters"], a["iters"] + 1, 200):
        b = P.solve(f, tol=1e-10, restart=m)
        assert b["iters"] == a["iters"] and b["mg_cycles_total"] == a["mg_cycles_total"]
        assert np.array_equal(b["u"], a["u"]) and np.array_equal(b["hist"], a["hist"])


def test_each_cycle_minimises_the_residual_over_its_krylov_space():
    # N = 8: 49 unknowns; one corner V-cycle per application, so M^{-1} is linear
    for name, eps in (("cfg4", 1e-8), ("cfg2", 1e-2), ("cfg5", 1e-2)):
        cfg, f, P = _mk(name, 8, eps, mg_fixed=1)
        n = P.m * P.m
        A = _cols(lambda v: P.matvec(v.reshape(P.m, P.m)), n)
        Minv = _cols(lambda v: P.precond(v.reshape(P.m, P.m)), n)
        D = P.coef()["D"].ravel()
        W = 1.0 / D
        B = (W[:, None] * A) @ Minv @ np.diag(D)
        fv = np.asarray(f).ravel()
        for m in (1, 2, 3):
            x = np.zeros(n)
            for cyc in range(3):
                rc = W * (fv - A @ x)
                K = np.empty((n, m))
                K[:, 0] = rc
                for j in range(1, m):
                    K[:, j] = B @ K[:, j - 1]
                Q, _ = np.linalg.qr(K)
                t = np.linalg.lstsq(B @ Q, rc, rcond=None)[0]
                x = x + Minv @ (D * (Q @ t))
                got = P.solve(f, tol=1e-300, maxit=m * (cyc + 1), fixed_iters=m * (cyc + 1), restart=m)
                assert got["iters"] == m * (cyc + 1)
                u = np.asarray(got["u"]).ravel()
                assert np.linalg.norm(u - x) <= 1e-10 * np.linalg.norm(x), (name, m, cyc)


def test_restarted_residual_history_is_monotone_and_converges():
    # cfg5 at eps = 1e-2 (eps N outside the method's regime, many iterations): FGMRES(5)
    cfg, f, P = _mk("cfg5", 64, 1e-2)
    full = P.solve(f, tol=1e-8, maxit=300)
    res = P.solve(f, tol=1e-8, maxit=300, restart=5)
    assert full["converged"] and res["converged"]
    assert res["iters"] >= full["iters"]          # restarting can only slow GMRES down
    h = res["hist"]
    assert np.all(h[1:] <= h[:-1] * (1 + 1e-10))   # each cycle starts from the true residual
    # the restarted iterate solves the same system (to the tolerance, Jacobi-weighted)
    ref = P.direct(f)
    assert np.linalg.norm(res["u"] - ref) <= 1e-6 * np.linalg.norm(ref)

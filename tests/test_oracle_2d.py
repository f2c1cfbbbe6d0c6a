"""Pins for the 2D oracle: 5-point upwind stencil, the block preconditioner of eq:2D blocks,
the corner multigrid and FGMRES, against what PAPER.md fixes (cited), closed forms,
invariants and numpy brute force on small meshes.  No expected value comes from the oracle
itself or from the CUDA path.
"""
import numpy as np
import pytest

import oracle
import spp_inputs as si
from conftest import load_table, rounds_to


def _mk(name, N, eps=None, sigma=2.0, bx=1.0, by=1.0, **kw):
    cfg = si.config(name, N=N, eps=eps)
    x = oracle.mesh(N, cfg.eps, sigma, bx)
    y = oracle.mesh(N, cfg.eps, sigma, by)
    c1, c2, r, f = si.sample_2d(cfg, x, y)
    P = oracle.Oracle2D(N, cfg.eps, x, y, c1, c2, r, **kw)
    return cfg, x, y, (c1, c2, r, f), P


def _exp2d(N, eps, **kw):
    return _mk("exp2d", N, eps, sigma=2.5, bx=1.99, by=2.99, **kw)   # reading R1


def _dense(P):
    m = P.m
    A = np.zeros((m * m, m * m))
    for k in range(m * m):
        e = np.zeros(m * m); e[k] = 1.0
        A[:, k] = P.matvec(e).ravel()
    return A


def _region(i, j, n):
    if i <= n and j <= n:
        return 0  # C
    if i <= n:
        return 1  # X
    if j <= n:
        return 2  # Y
    return 3      # I


def _mhat(A, N):
    """M-hat of P:1113-1116 built from A by the block rules of eq:2D blocks:
    upper blocks kept, lower blocks dropped; diagonal blocks: C exact; X keeps its lines
    (constant y) and the North neighbour; Y keeps its lines (constant x) and the East
    neighbour; I keeps the diagonal, East and North (upper-triangular part)."""
    m, n = N - 1, N // 2
    M = np.zeros_like(A)
    for p in range(m * m):
        jp, ip = divmod(p, m); ip += 1; jp += 1
        rp = _region(ip, jp, n)
        for q in np.nonzero(A[p])[0]:
            jq, iq = divmod(q, m); iq += 1; jq += 1
            rq = _region(iq, jq, n)
            keep = False
            if rp < rq:
                keep = True
            elif rp == rq:
                di, dj = iq - ip, jq - jp
                if rp == 0:
                    keep = True
                elif rp == 1:      # X: same line (dj == 0) or North
                    keep = dj == 0 or dj == 1
                elif rp == 2:      # Y: same line (di == 0) or East
                    keep = di == 0 or di == 1
                else:              # I: diagonal, East, North
                    keep = (di, dj) in ((0, 0), (1, 0), (0, 1))
            if keep:
                M[p, q] = A[p, q]
    return M


# ---------------------------------------------------------------- operator
def test_uniform_mesh_stencil_closed_form():
    """eps = 1 clamps tau to 1/2 (uniform mesh h = 1/N): the stencil of P:972-981 becomes
    W = -eps N^2, E = -eps N^2 - c1 N, S = -eps N^2, N = -eps N^2 - c2 N,
    centre = 4 eps N^2 + (c1 + c2) N + r."""
    N = 8
    cfg = si.config("cfg5", N=N, eps=1.0)
    x = oracle.mesh(N, 1.0, 2.0, 1.0)
    c1 = np.full((N - 1, N - 1), 1.3); c2 = np.full_like(c1, 0.7); r = np.full_like(c1, 0.4)
    P = oracle.Oracle2D(N, 1.0, x, x, c1, c2, r)
    A = _dense(P)
    m = N - 1
    p = (3 - 1) * m + (4 - 1)          # node (i=4, j=3)
    assert np.isclose(A[p, p], 4 * N**2 + 2.0 * N + 0.4, rtol=1e-14)
    assert np.isclose(A[p, p - 1], -N**2, rtol=1e-14)
    assert np.isclose(A[p, p + 1], -N**2 - 1.3 * N, rtol=1e-14)
    assert np.isclose(A[p, p - m], -N**2, rtol=1e-14)
    assert np.isclose(A[p, p + m], -N**2 - 0.7 * N, rtol=1e-14)
    assert np.count_nonzero(A[p]) == 5
    del cfg


@pytest.mark.parametrize("eps", [1e-2, 1e-6, 1e-10])
def test_m_matrix_sign_pattern_and_row_sums(eps):
    """irreducibly diagonally dominant M-matrix; A*1 = r on rows not touching the
    boundary (exactly, in difference form)."""
    N = 16
    _, x, y, (c1, c2, r, f), P = _mk("cfg4", N, eps)
    A = _dense(P)
    d = np.diag(A)
    off = A - np.diag(d)
    assert np.all(d > 0) and np.all(off <= 0)
    assert np.all(np.abs(off).sum(1) <= d)
    y1 = P.matvec(np.ones((N - 1, N - 1)))
    assert np.array_equal(y1[1:-1, 1:-1], r[1:-1, 1:-1])
    # barrier function of P:1148-1153.  For -c.grad u with c1 > 0 the printed W = 1 + x_i gives
    # A W = -c1 + r(1+x); the barrier that works is W = 2 - x_i (A W >= min c1): DESIGN.md R19.
    W = np.tile(2 - x[1:-1], (N - 1, 1))
    assert np.all(P.matvec(W) >= c1.min() * (1 - 1e-12))


def test_direct_solve_brute_force():
    N = 16
    _, x, y, (c1, c2, r, f), P = _mk("cfg4", N, 1e-8)
    A = _dense(P)
    ue = np.linalg.solve(A, f.ravel())
    u = P.direct(f).ravel()
    assert np.linalg.norm(u - ue) <= 1e-12 * np.linalg.norm(ue)


# ---------------------------------------------------------------- preconditioner
@pytest.mark.parametrize("name,eps", [("cfg4", 1e-8), ("cfg3", 1e-6), ("cfg5", 1e-2), ("exp2d", 1e-5)])
def test_block_preconditioner_equals_dense_mhat(name, eps):
    """With the corner solved to rounding, M^{-1} q equals a dense solve with M-hat
    constructed independently from A by the rules of eq:2D blocks."""
    N = 16
    if name == "exp2d":
        _, x, y, ins, P = _exp2d(N, eps, mg_red=1e-14, mg_cap=400)
    else:
        _, x, y, ins, P = _mk(name, N, eps, mg_red=1e-14, mg_cap=400)
    A = _dense(P)
    Mh = _mhat(A, N)
    Nh = Mh - A
    assert np.all(Nh >= 0)                         # regular splitting
    q = si.random_field(11, (N - 1, N - 1))
    z = P.precond(q).ravel()
    zz = np.linalg.solve(Mh, q.ravel())
    assert np.linalg.norm(z - zz) <= 1e-11 * np.linalg.norm(zz)
    # rho(I - Mhat^{-1} A) < 1
    G = np.eye(A.shape[0]) - np.linalg.solve(Mh, A)
    assert np.max(np.abs(np.linalg.eigvals(G))) < 1


def test_stage_order_and_partial_solves():
    """Each stage solves its diagonal block with the already-computed neighbours on the
    rhs (block back-substitution of eq:2D blocks): check block rows of M-hat z = q."""
    N = 16
    _, x, y, ins, P = _mk("cfg4", N, 1e-8)
    A = _dense(P)
    Mh = _mhat(A, N)
    m, n = N - 1, N // 2
    q = si.random_field(12, (m, m))
    z = P.stage_I(q)
    z = P.stage_Y(q, z)
    z = P.stage_X(q, z)
    reg = np.array([_region(i, j, n) for j in range(1, N) for i in range(1, N)])
    res = (Mh @ z.ravel() - q.ravel())
    scale = np.abs(Mh) @ np.abs(z.ravel()) + np.abs(q.ravel())     # rounding scale per row
    for rg in (1, 2, 3):       # X, Y and I rows are solved exactly
        assert np.all(np.abs(res[reg == rg]) <= 1e-13 * scale[reg == rg])
    bC = P.corner_rhs(q, z)
    # b_C = q_C - A_CX z_X - A_CY z_Y
    AC = A[np.ix_(reg == 0, reg != 0)]
    want = q.ravel()[reg == 0] - AC @ z.ravel()[reg != 0]
    assert np.allclose(bC.ravel(), want, rtol=1e-13, atol=1e-14 * np.abs(want).max())


def _dense_level(P, l):
    nl = P.level_n(l)
    A = np.zeros((nl * nl, nl * nl))
    for k in range(nl * nl):
        e = np.zeros(nl * nl); e[k] = 1.0
        A[:, k] = -P.level_residual(l, np.zeros(nl * nl), e).ravel()
    return A


def test_corner_level0_is_A_CC():
    """Reading R8: with node n+1 kept as the block's Dirichlet node, the level-0 operator is
    A_CC itself (same coefficients, bit for bit)."""
    N = 32
    _, x, y, ins, P = _mk("cfg3", N, 1e-6)
    g, c0 = P.coef(), P.level_coef(0)
    n = N // 2
    assert np.array_equal(c0["aE"], g["aE"][:n, :n])
    assert np.array_equal(c0["aN"], g["aN"][:n, :n])
    assert np.array_equal(c0["D"], g["D"][:n, :n])
    assert np.array_equal(c0["aW"][1:n + 1], g["aW"][1:n + 1])
    assert np.array_equal(c0["aS"][1:n + 1], g["aS"][1:n + 1])
    A = _dense(P)
    reg = np.array([_region(i, j, n) for j in range(1, N) for i in range(1, N)])
    assert np.allclose(_dense_level(P, 0), A[np.ix_(reg == 0, reg == 0)], rtol=1e-14, atol=0)
    assert P.levels == 3 and [P.level_n(l) for l in range(3)] == [16, 8, 4]   # coarsest <= 4


@pytest.mark.parametrize("l", [0, 1])
def test_gs_sweep_is_downstream_triangular_solve(l):
    """downstream point GS from the top-right to the bottom-left point:
    e_new = (D - E - N)^{-1} (b + (W + S) e_old) with the splitting of A_l by direction."""
    N = 32
    _, x, y, ins, P = _mk("cfg4", N, 1e-8)
    Al = _dense_level(P, l)
    nl = P.level_n(l)
    up = np.zeros_like(Al)
    for p in range(nl * nl):
        for q in np.nonzero(Al[p])[0]:
            if q == p or q == p + 1 and (p % nl) != nl - 1 or q == p + nl:
                up[p, q] = Al[p, q]
    low = up - Al
    b = si.random_field(21, (nl, nl)).ravel()
    e0 = si.random_field(22, (nl, nl)).ravel()
    e1 = P.gs_sweep(l, b, e0).ravel()
    want = np.linalg.solve(up, b + low @ e0)
    assert np.linalg.norm(e1 - want) <= 1e-12 * np.linalg.norm(want)


def test_transfer_operators():
    """restriction is S_c^{-1} P^T S_f with P bilinear (weights 1, 1/2, 1/4):
    adjointness <P e_c, S_f v> = <e_c, S_c R v>, and P reproduces bilinear functions that
    vanish on the Dirichlet side."""
    N = 32
    _, x, y, ins, P = _mk("cfg5", N, 1e-6)
    f0, c1 = P.level_coef(0), P.level_coef(1)
    nf, nc = f0["n"], c1["n"]
    Sf = np.outer(f0["kb"][1:nf + 1], f0["hb"][1:nf + 1])
    Sc = np.outer(c1["kb"][1:nc + 1], c1["hb"][1:nc + 1])
    v = si.random_field(31, (nf, nf))
    ec = si.random_field(32, (nc, nc))
    Pe = P.prolong_add(0, ec, np.zeros((nf, nf)))
    Rv = P.restrict(0, v)
    assert np.isclose(np.sum(Pe * Sf * v), np.sum(ec * Sc * Rv), rtol=1e-13)
    I = np.arange(1, nf + 1)
    lin = np.outer(I, 2 * I) * 1.0                      # bilinear in the fine index, 0 at 0
    Ic = np.arange(1, nc + 1)
    linc = np.outer(2 * Ic, 4 * Ic) * 1.0               # same function at coarse nodes
    assert np.allclose(P.prolong_add(0, linc, np.zeros((nf, nf))), lin, rtol=1e-15)
    # interpolation weights on a single coarse impulse: 1, 1/2, 1/4
    imp = np.zeros((nc, nc)); imp[2, 3] = 1.0           # coarse (I=4, J=3) -> fine (8, 6)
    Pi = P.prolong_add(0, imp, np.zeros((nf, nf)))
    assert Pi[5, 7] == 1.0 and Pi[5, 6] == 0.5 and Pi[4, 7] == 0.5 and Pi[4, 6] == 0.25
    assert np.count_nonzero(Pi) == 9


@pytest.mark.parametrize("name,eps", [("cfg4", 1e-8), ("cfg2", 1e-2), ("exp2d", 1e-4)])
def test_corner_mg_converges_to_dense_solve(name, eps):
    N = 32
    if name == "exp2d":
        _, x, y, ins, P = _exp2d(N, eps, mg_red=1e-14, mg_cap=200)
    else:
        _, x, y, ins, P = _mk(name, N, eps, mg_red=1e-14, mg_cap=200)
    n = N // 2
    b = si.random_field(41, (n, n))
    z, cyc, cap = P.corner_solve(b)
    AC = _dense_level(P, 0)
    zz = np.linalg.solve(AC, b.ravel())
    assert not cap
    assert np.linalg.norm(z.ravel() - zz) <= 1e-12 * np.linalg.norm(zz)
    # r = 0 -> z = 0, zero cycles
    z0, c0, _ = P.corner_solve(np.zeros((n, n)))
    assert c0 == 0 and not np.any(z0)


def test_vcycle_linear():
    """the V-cycle is linear: V(10 b) = 10 V(b)."""
    N = 64
    _, x, y, ins, P = _mk("cfg4", N, 1e-8)
    b = si.random_field(51, (N // 2, N // 2))
    e1, e10 = P.vcycle(0, b), P.vcycle(0, 10 * b)
    assert np.allclose(e10, 10 * e1, rtol=1e-13, atol=1e-13 * np.abs(e10).max())


# ---------------------------------------------------------------- Tables 6 and 7
T6 = load_table("table6_exp_errors.txt")
T7 = load_table("table7_exp_iters.txt")


@pytest.mark.parametrize("col,N", [(0, 128), (1, 256), (2, 512), (3, 1024)])
def test_tables_6_7_exponential(col, N):
    """FGMRES counts (exact) and max-norm errors (4 digits) for
    eq:exponential_MMS, sigma = 5/2, stop ||R||_2 <= 10 N^{-1} ln N; and the corner MG takes
    5 cycles per apply."""
    for eps in sorted(T7):
        cfg, x, y, (c1, c2, r, f), P = _exp2d(N, eps)
        res = P.solve(f, weighted=0, stop_abs=1, tol=cfg.tol, maxit=100)
        assert res["iters"] == int(T7[eps][col]), (N, eps, res["iters"])
        err = np.max(np.abs(res["u"] - si.exact_solution(cfg, x, y)))
        assert rounds_to(err, T6[eps][col]), (eps, N, err, T6[eps][col])
        assert set(res["cycle_log"]) == {5}
        P.close()


# ---------------------------------------------------------------- BASELINE workloads
def test_cfg2_first_order_convergence():
    """B:8 with the corrected factor (reading R13): U^E -> u* at the almost-first-order rate
    N^{-1} ln N of the Shishkin-mesh upwind scheme (eq:error bound 1D Shishkin analogue)."""
    errs = []
    for N in (64, 128):
        cfg, x, y, (c1, c2, r, f), P = _mk("cfg2", N)
        u = P.direct(f)
        errs.append(np.max(np.abs(u - si.exact_solution(cfg, x, y))))
    rate = (np.log(64) / 64) / (np.log(128) / 128)
    assert 0.8 * rate <= errs[0] / errs[1] <= 1.2 * rate
    assert errs[1] <= np.log(128) / 128


@pytest.mark.parametrize("name,eps", [("cfg4", 1e-8), ("cfg5", 1e-10), ("cfg3", 1e-6), ("cfg5", 1e-2)])
def test_fgmres_deep_check_vs_direct(name, eps):
    """O2 at rtol 1e-12 (Jacobi-weighted) agrees with O1 (banded LU + difference-form
    refinement); the recurrence residual equals the true weighted residual; monotone."""
    N = 64
    cfg, x, y, (c1, c2, r, f), P = _mk(name, N, eps)
    res = P.solve(f, weighted=1, tol=1e-12, maxit=200)
    ue = P.direct(f)
    assert res["converged"]
    assert np.linalg.norm(res["u"] - ue) <= 2e-10 * np.linalg.norm(ue)
    D = P.coef()["D"]
    true_rel = np.linalg.norm((f - P.matvec(res["u"])) / D) / np.linalg.norm(f / D)
    rec_rel = res["hist"][-1] / res["hist"][0]
    assert true_rel <= 1e-11 and abs(true_rel - rec_rel) <= 1e-3 * max(rec_rel, 1e-14) + 1e-14
    assert np.all(np.diff(res["hist"]) <= 1e-12 * res["hist"][0])


def test_baseline_iteration_counts_small_eps_robust():
    """eps-robustness (B:5): at small eps the Jacobi-weighted iteration count is flat in
    eps and N (cfg4 proxies take 3 iterations)."""
    its = []
    for N in (128, 256):
        for eps in (1e-6, 1e-8, 1e-10):
            cfg, x, y, (c1, c2, r, f), P = _mk("cfg4", N, eps)
            its.append(P.solve(f, weighted=1, tol=1e-8, maxit=100)["iters"])
    assert max(its) - min(its) <= 1 and max(its) <= 4


def test_fgmres_nonfinite_guard():
    """SURVEY 5 "NaN/Inf guard on h_{k+1,k}": a NaN right-hand side is an error (rc -10), not a
    breakdown reported as convergence."""
    import pytest
    N, eps = 16, 1e-3
    x = oracle.mesh(N, eps)
    m = N - 1
    P = oracle.Oracle2D(N, eps, x, x, np.ones(m * m), np.ones(m * m), np.ones(m * m))
    f = np.ones(m * m)
    f[7] = np.nan
    with pytest.raises(RuntimeError, match="rc=-10"):
        P.solve(f, weighted=1, tol=1e-8)
    f[7] = np.inf
    with pytest.raises(RuntimeError, match="rc=-10"):
        P.solve(f, weighted=0, tol=1e-8)
    # an exact zero rhs is not an error: x = 0 after zero iterations
    res = P.solve(np.zeros(m * m), weighted=1, tol=1e-8)
    assert res["iters"] == 0 and res["converged"]

"""Pins for the 1D oracle (mesh, eq:stencil_1d, eq:block_M, GMRES) against what the paper fixes.

Every expected value here is printed in PAPER.md / SPEC.md (cited) or is a closed form,
an invariant or a library (numpy) brute-force solve -- never a value produced by the oracle
itself or by the CUDA path.
"""
import numpy as np
import pytest

import oracle
import spp_inputs as si
from conftest import load_table, rounds_to

CL = 0.99   # reading R1: C_lower = min c - 0.01; pinned by Table 1 below


def _ex1d(N, eps):
    cfg = si.config("ex1d", N=N, eps=eps)
    x = oracle.mesh(N, eps, 2.0, CL)
    c, r, f = si.sample_1d(cfg, x)
    return cfg, x, c, r, f


def _fine_mesh(tau, Nf):
    """Benchmark mesh of P:737-741: same transition point, Nf intervals (Nf/2 per side)."""
    n = Nf // 2
    return np.concatenate([np.arange(n) * (tau / n), [tau],
                           tau + np.arange(1, n) * ((1 - tau) / n), [1.0]])


def _dense(N, eps, x, c, r):
    m = N - 1
    A = np.zeros((m, m))
    for k in range(m):
        e = np.zeros(m); e[k] = 1.0
        A[:, k] = oracle.matvec1d(N, eps, x, c, r, e)
    return A


# ---------------------------------------------------------------- mesh (eq:tau 1D)
def test_mesh_spec_examples():
    # (eps=1e-8, N=128, C=1) -> tau ~ 9.70406e-8, h_1 ~ 1.51626e-9, h_N ~ 1.5625e-2
    x = oracle.mesh(128, 1e-8, 2.0, 1.0)
    assert abs(x[64] / 9.70406e-8 - 1) < 1e-6
    assert abs((x[1] - x[0]) / 1.51626e-9 - 1) < 1e-5
    assert abs((x[128] - x[127]) / 1.5625e-2 - 1) < 1e-6
    # eps = 1 clamps tau to 1/2 -> uniform mesh
    x = oracle.mesh(128, 1.0, 2.0, 1.0)
    assert np.allclose(np.diff(x), 1 / 128, rtol=0, atol=1e-15)
    # (eps=1e-6, N=256, sigma=5/2, C1=2, C2=3) -> tau_x ~ 6.93147e-6, tau_y ~ 4.62098e-6
    assert abs(oracle.mesh(256, 1e-6, 2.5, 2.0)[128] / 6.93147e-6 - 1) < 1e-6
    assert abs(oracle.mesh(256, 1e-6, 2.5, 3.0)[128] / 4.62098e-6 - 1) < 1e-6


@pytest.mark.parametrize("N,eps", [(8, 1e-3), (256, 1e-4), (1024, 1e-10)])
def test_mesh_piecewise_uniform(N, eps):
    x = oracle.mesh(N, eps, 2.0, 1.0)
    tau = min(0.5, 2 * eps * np.log(N))          # closed form eq:tau 1D with C = 1
    assert x[0] == 0.0 and x[N] == 1.0 and x[N // 2] == tau
    h = np.diff(x)
    assert np.all(h > 0)
    assert np.allclose(h[: N // 2], tau / (N // 2), rtol=1e-9)
    assert np.allclose(h[N // 2:], (1 - tau) / (N // 2), rtol=1e-9)


def test_mesh_rejects_bad_input():
    for args in [(7, 1e-3, 2.0, 1.0), (2, 1e-3, 2.0, 1.0), (8, 0.0, 2.0, 1.0), (8, 2.0, 2.0, 1.0)]:
        with pytest.raises(ValueError):
            oracle.mesh(*args)


# ---------------------------------------------------------------- operator (eq:stencil_1d)
def test_uniform_mesh_stencil_closed_form():
    # on a uniform mesh h = 1/N the stencil is [-eps N^2, 2 eps N^2 + c N + r, -eps N^2 - c N]
    N, eps, c0, r0 = 32, 1.0, 1.7, 0.3
    x = oracle.mesh(N, eps, 2.0, 1.0)             # tau clamps to 1/2: uniform
    c, r = np.full(N - 1, c0), np.full(N - 1, r0)
    A = _dense(N, eps, x, c, r)
    m = N - 1
    assert np.allclose(np.diag(A), 2 * eps * N**2 + c0 * N + r0, rtol=1e-13)
    assert np.allclose(np.diag(A, -1), -eps * N**2, rtol=1e-13)
    assert np.allclose(np.diag(A, 1), -eps * N**2 - c0 * N, rtol=1e-13)
    assert np.count_nonzero(A) == 3 * m - 2


@pytest.mark.parametrize("eps", [1.0, 1e-2, 1e-4, 1e-8])
def test_m_matrix_and_row_sums(eps):
    # an M-matrix for any eps and mesh; A*1 = r away from the boundary
    N = 64
    _, x, c, r, _ = _ex1d(N, eps)
    A = _dense(N, eps, x, c, r)
    off = A - np.diag(np.diag(A))
    assert np.all(np.diag(A) > 0) and np.all(off <= 0)
    rs = A @ np.ones(N - 1)
    assert np.allclose(rs[1:-1], r[1:-1], rtol=0, atol=1e-12 * np.abs(A).max())
    assert np.all(rs >= r - 1e-12 * np.abs(A).max())
    # exact in difference form: the oracle's matvec of a constant returns r on interior rows
    y = oracle.matvec1d(N, eps, x, c, r, np.ones(N - 1))
    assert np.array_equal(y[1:-1], r[1:-1])


def test_direct_solve_brute_force():
    N, eps = 32, 1e-5
    _, x, c, r, f = _ex1d(N, eps)
    A = _dense(N, eps, x, c, r)
    ue = np.linalg.solve(A, f)
    u = oracle.direct1d(N, eps, x, c, r, f)
    assert np.linalg.norm(u - ue) <= 1e-13 * np.linalg.norm(ue)


def test_thomas_spec_examples():
    # tri(-1,2,-1), rhs e1 -> (3/4, 1/2, 1/4);  S:268 identity
    assert np.allclose(oracle.thomas([0, -1, -1], [2, 2, 2], [-1, -1, 0], [1, 0, 0]), [0.75, 0.5, 0.25])
    b = np.array([3.0, -1.0, 2.0])
    assert np.array_equal(oracle.thomas([0, 0, 0], [1, 1, 1], [0, 0, 0], b), b)
    rng = np.random.default_rng(5)
    for _ in range(10):
        m = 100
        lo, up = -rng.random(m), -rng.random(m)
        di = 2.5 + rng.random(m)
        rhs = rng.standard_normal(m)
        T = np.diag(di) + np.diag(lo[1:], -1) + np.diag(up[:-1], 1)
        assert np.allclose(oracle.thomas(lo, di, up, rhs), np.linalg.solve(T, rhs), rtol=1e-11, atol=1e-12)


# ---------------------------------------------------------------- Table 1 (discretisation)
T1 = load_table("table1_1d_errors.txt")


@pytest.mark.parametrize("eps", sorted(T1))
def test_table1_errors(eps):
    """max-norm error vs the 64N benchmark, 4 printed digits."""
    for col, N in enumerate([128, 256, 512]):
        _, x, c, r, f = _ex1d(N, eps)
        u = oracle.direct1d(N, eps, x, c, r, f)
        Nf = 64 * N
        xf = _fine_mesh(x[N // 2], Nf)
        cf, rf, ff = si.sample_1d(si.config("ex1d", N=Nf, eps=eps), xf)
        uf = oracle.direct1d(Nf, eps, xf, cf, rf, ff)
        err = np.max(np.abs(u - uf[63::64][: N - 1]))
        assert rounds_to(err, T1[eps][col]), (eps, N, err, T1[eps][col])


# ---------------------------------------------------------------- preconditioner theory
@pytest.mark.parametrize("eps", [1e-4, 1e-6, 1e-8])
def test_theorem_block_fact_unit_eigenvectors(eps):
    """Theorem block_fact: (M^{-1}A) e_k = e_k for k <= N_L."""
    N = 128
    _, x, c, r, _ = _ex1d(N, eps)
    m, NL = N - 1, N // 2
    for k in range(NL):
        e = np.zeros(m); e[k] = 1.0
        z = oracle.precond1d(N, eps, x, c, r, oracle.matvec1d(N, eps, x, c, r, e))
        assert np.max(np.abs(z - e)) <= 1e-12


def test_preconditioner_structure_brute_force():
    """eq:block_M: M = A with A_II replaced by its upper triangle (diagonal kept)."""
    N, eps = 32, 1e-6
    _, x, c, r, _ = _ex1d(N, eps)
    A = _dense(N, eps, x, c, r)
    NL = N // 2
    M = A.copy()
    # rows/cols NL+1..N-1 (1-based) form A_II; keep its upper triangle
    I = slice(NL, N - 1)
    M[I, I] = np.triu(A[I, I])
    q = si.random_field(3, (N - 1,))
    z = oracle.precond1d(N, eps, x, c, r, q)
    assert np.linalg.norm(z - np.linalg.solve(M, q)) <= 1e-12 * np.linalg.norm(z)


@pytest.mark.parametrize("eps,N", [(1e-6, 128), (1e-5, 128), (1e-6, 256)])
def test_spectral_band(eps, N):
    """Theorem big_bound and the observed band of P:773-779:
    1 - 4 eps N/(C alpha) <= lambda_min <= 1 - eps N /(2 C alpha),  alpha = 2(1 - 2 eps ln N / C)."""
    _, x, c, r, _ = _ex1d(N, eps)
    A = _dense(N, eps, x, c, r)
    m = N - 1
    Minv_A = np.column_stack([oracle.precond1d(N, eps, x, c, r, A[:, k]) for k in range(m)])
    # Theorem block_fact: M^{-1}A = [[I, *], [0, S_M^{-1} S_A]] in this basis; the non-unit
    # eigenvalues are those of the trailing block (avoids the defective unit cluster).
    NL = N // 2
    assert np.allclose(Minv_A[NL:, :NL], 0, atol=1e-12)
    lam = np.linalg.eigvals(Minv_A[NL:, NL:])
    alpha = 2 * (1 - 2 * eps * np.log(N) / CL)
    lmin = lam.real.min()
    assert lmin >= 1 - 8 * eps * N / (CL * alpha) - 1e-9          # theorem
    assert 1 - 4 * eps * N / (CL * alpha) <= lmin <= 1 - eps * N / (2 * CL * alpha)
    # eigenvalues <= 1 (theorem); the cluster at 1 is defective, so allow eigen-solver noise
    assert lam.real.max() <= 1 + 1e-4


# ---------------------------------------------------------------- Table 2 (GMRES counts)
T2 = load_table("table2_1d_iters.txt")


@pytest.mark.parametrize("eps", sorted(T2))
def test_table2_iteration_counts(eps):
    """left-preconditioned GMRES, no restarts, ||b-Ax||_inf <= N^{-1} ln N (K=1)."""
    for col, N in enumerate([128, 256, 512, 1024, 2048]):
        want = T2[eps][col]
        if want is None:
            continue
        _, x, c, r, f = _ex1d(N, eps)
        res = oracle.solve1d(N, eps, x, c, r, f, side=1, tol=np.log(N) / N, maxit=200)
        assert res["iters"] == int(want), (eps, N, res["iters"], want)


def test_gmres_right_weighted_matches_direct():
    """BASELINE mode (right/flexible, Jacobi-weighted recurrence stop) at a tight tolerance
    reaches the exact discrete solution; recurrence residual equals the true weighted one."""
    cfg = si.config("cfg1")
    N, eps = cfg.N, cfg.eps
    x = oracle.mesh(N, eps, 2.0, 1.0)
    c, r, f = si.sample_1d(cfg, x)
    res = oracle.solve1d(N, eps, x, c, r, f, side=0, weighted=1, tol=1e-13, maxit=100)
    ue = oracle.direct1d(N, eps, x, c, r, f)
    assert np.linalg.norm(res["u"] - ue) <= 1e-11 * np.linalg.norm(ue)
    A = _dense(N, eps, x, c, r)
    D = np.diag(A)
    true_rel = np.linalg.norm((f - A @ res["u"]) / D) / np.linalg.norm(f / D)
    assert true_rel <= 1e-12
    assert np.all(np.diff(res["hist"]) <= 1e-12 * res["hist"][0])      # monotone


def test_gmres_identity_one_step():
    """A = I (eps tiny is irrelevant) -- use the 1D driver with M = A exactly:
    when N_I <= 1 the preconditioner equals A and GMRES converges in one step."""
    N, eps = 4, 1e-3         # N_L = 2, I = {3}: M = A
    x = oracle.mesh(N, eps, 2.0, 1.0)
    c, r, f = np.ones(3), np.ones(3), np.array([1.0, -2.0, 0.5])
    res = oracle.solve1d(N, eps, x, c, r, f, side=0, weighted=0, tol=1e-12, maxit=10)
    assert res["iters"] == 1

"""Graded layer-adapted meshes on the GPU (R21): Bakhvalov-Shishkin
meshes through the same kernels (coordinate-difference widths, corner levels with geometric
interpolation weights) against the oracle on the same seeded inputs -- identical FGMRES and
corner-cycle counts, solutions within 1e-9 relative l2 -- plus the transfer kernels through the
product-path hooks, the row strips, and several right-hand sides per setup."""
import numpy as np
import pytest

import oracle
import spp_inputs as si

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2108_13468_b200 as spp  # noqa: E402


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64).ravel()).cuda()


def rel(a, b):
    a, b = np.asarray(a).ravel(), np.asarray(b).ravel()
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def relmax(a, b):
    a, b = np.asarray(a).ravel(), np.asarray(b).ravel()
    return np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300)


def _bs(name, N, eps, sigma=2.0, bx=1.0, by=1.0, stop=spp.SPP_STOP_REL_JACOBI, strips=1, **opt):
    cfg = si.config(name, N=N, eps=eps)
    x = spp.spp_bakhvalov_mesh(N, cfg.eps, sigma, bx)
    y = spp.spp_bakhvalov_mesh(N, cfg.eps, sigma, by)
    assert np.array_equal(x, oracle.mesh_bs(N, cfg.eps, sigma, bx))
    c1, c2, r, f = si.sample_2d(cfg, x, y)
    o = spp.spp_default_options(2)
    o.stop, o.tol = stop, cfg.tol
    for k, v in opt.items():
        setattr(o, k, v)
    S = spp.Solver(2, N, cfg.eps, x, y, dev(c1), dev(c2), dev(r), options=o, strips=strips)
    P = oracle.Oracle2D(N, cfg.eps, x, y, c1, c2, r, mg_red=o.mg_reduction, mg_cap=o.mg_max_cycles,
                        mg_fixed=o.mg_fixed_cycles)
    return cfg, x, y, (c1, c2, r, f), S, P, o


@pytest.mark.parametrize("name,N,eps", [("cfg4", 256, 1e-8), ("cfg4", 1024, 1e-8), ("cfg4", 512, 1e-4),
                                        ("cfg5", 512, 1e-6), ("cfg3", 512, 1e-6), ("cfg2", 128, 1e-2)])
def test_bs_solve_matches_oracle(name, N, eps):
    cfg, x, y, (c1, c2, r, f), S, P, o = _bs(name, N, eps)
    res = S.solve(dev(f))
    ores = P.solve(f, weighted=1, tol=o.tol, maxit=o.max_iters)
    assert res.stats["iters"] == ores["iters"], (res.stats["iters"], ores["iters"])
    assert res.stats["mg_cycles_total"] == ores["mg_cycles_total"]
    assert res.stats["mg_cap_hits"] == ores["mg_cap_hits"]
    assert rel(res.u.cpu().numpy(), ores["u"]) <= 1e-9
    np.testing.assert_allclose(res.hist, ores["hist"], rtol=1e-6, atol=1e-14 * ores["hist"][0])


@pytest.mark.parametrize("N", [128, 256])
def test_bs_paper_workload(N):
    """eq:exponential_MMS in paper mode on Bakhvalov-Shishkin meshes: the GPU
    reproduces the oracle's counts and error, and the error is below the Shishkin mesh's at the same
    N (the N^{-1} rate without the ln N factor, tests/test_oracle_bs.py)."""
    eps = 1e-6
    cfg, x, y, (c1, c2, r, f), S, P, o = _bs("exp2d", N, eps, sigma=2.5, bx=1.99, by=2.99, stop=spp.SPP_STOP_ABS_L2)
    res = S.solve(dev(f))
    ores = P.solve(f, weighted=0, stop_abs=1, tol=o.tol, maxit=o.max_iters)
    u = res.u.cpu().numpy()
    assert res.stats["iters"] == ores["iters"] and res.stats["mg_cycles_total"] == ores["mg_cycles_total"]
    assert rel(u, ores["u"]) <= 1e-9
    err = np.max(np.abs(u.reshape(N - 1, N - 1) - si.exact_solution(cfg, x, y)))
    xs = spp.spp_shishkin_mesh(N, eps, 2.5, 1.99)
    ys = spp.spp_shishkin_mesh(N, eps, 2.5, 2.99)
    cs = si.sample_2d(cfg, xs, ys)
    Ss = spp.Solver(2, N, eps, xs, ys, dev(cs[0]), dev(cs[1]), dev(cs[2]), options=o)
    us = Ss.solve(dev(cs[3])).u.cpu().numpy()
    err_s = np.max(np.abs(us.reshape(N - 1, N - 1) - si.exact_solution(cfg, xs, ys)))
    assert err < err_s


def test_bs_transfer_hooks():
    """The fused residual-restriction and prolongation-smoothing kernels with the geometric
    interpolation weights of a graded corner, against the oracle's definitions."""
    cfg, x, y, ins, S, P, o = _bs("cfg5", 256, 1e-6, by=2.0)
    for l in range(P.levels - 1):
        nl, nc = P.level_n(l), P.level_n(l + 1)
        b = si.random_field(70 + l, (nl, nl))
        e0 = si.random_field(80 + l, (nl, nl))
        ec = si.random_field(90 + l, (nc, nc))
        out = torch.zeros(nl * nl, dtype=torch.float64, device="cuda")
        S.apply_stage("POST_SMOOTH", torch.cat([dev(b), dev(e0), dev(ec)]), out, level=l)
        assert relmax(out.cpu().numpy(), P.gs_sweep(l, b, P.prolong_add(l, ec, e0))) <= 1e-12, l
        out = torch.zeros(nc * nc, dtype=torch.float64, device="cuda")
        S.apply_stage("RESID_RESTRICT", torch.cat([dev(b), dev(e0)]), out, level=l)
        want = P.restrict(l, P.level_residual(l, b, e0)) / P.level_coef(l + 1)["D"]
        assert relmax(out.cpu().numpy(), want) <= 1e-12, l
        out = torch.zeros(nc * nc, dtype=torch.float64, device="cuda")
        S.apply_stage("PRE_RESTRICT", dev(b), out, level=l)
        e1 = P.gs_sweep(l, b, np.zeros((nl, nl)))
        want = P.restrict(l, P.level_residual(l, b, e1)) / P.level_coef(l + 1)["D"]
        assert relmax(out.cpu().numpy(), want) <= 1e-12, l
        out = dev(e0)
        S.apply_stage("PROLONG_ADD", dev(ec), out, level=l)
        assert relmax(out.cpu().numpy(), P.prolong_add(l, ec, e0)) <= 1e-14, l
    nl = P.level_n(P.levels - 1)
    b = si.random_field(99, (P.level_n(0),) * 2)
    out = torch.zeros(b.size, dtype=torch.float64, device="cuda")
    S.apply_stage("VCYCLE", dev(b), out, level=0)
    assert relmax(out.cpu().numpy(), P.vcycle(0, b)) <= 1e-11
    del nl


def test_bs_row_strips():
    cfg, x, y, (c1, c2, r, f), S1, P, o = _bs("cfg4", 512, 1e-8)
    r1 = S1.solve(dev(f))
    S4 = spp.Solver(2, 512, cfg.eps, x, y, dev(c1), dev(c2), dev(r), options=o, strips=4)
    r4 = S4.solve(dev(f))
    assert r4.stats["iters"] == r1.stats["iters"] and r4.stats["mg_cycles_total"] == r1.stats["mg_cycles_total"]
    assert rel(r4.u.cpu().numpy(), r1.u.cpu().numpy()) <= 1e-12


@pytest.mark.parametrize("mesh", ["shishkin", "bakhvalov"])
def test_several_right_hand_sides_per_setup(mesh):
    """NEXT-4's other half: one setup (coefficients, line factors, multigrid levels) serves any
    number of right-hand sides; each solve equals a fresh create + solve bit for bit."""
    N, eps = 256, 1e-8
    cfg = si.config("cfg4", N=N, eps=eps)
    mk = spp.spp_shishkin_mesh if mesh == "shishkin" else spp.spp_bakhvalov_mesh
    x = mk(N, eps)
    c1, c2, r, f = si.sample_2d(cfg, x, x)
    S = spp.Solver(2, N, eps, x, x, dev(c1), dev(c2), dev(r))
    for k in range(3):
        fk = f + k * si.random_field(300 + k, f.shape)
        uk = S.solve(dev(fk)).u.cpu().numpy()
        Sf = spp.Solver(2, N, eps, x, x, dev(c1), dev(c2), dev(r))
        assert np.array_equal(uk, Sf.solve(dev(fk)).u.cpu().numpy())
        Sf.close()

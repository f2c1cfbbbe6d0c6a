"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the same seeded
inputs.  Bars (BASELINE north_star, B:5): fp64 solutions within 1e-9 relative l2 of the
oracle's iterate, iteration counts within +-1 (identical expected); single kernels within
the rounding bounds stated per test."""
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


def host(t):
    return t.cpu().numpy()


def rel(a, b):
    a, b = np.asarray(a).ravel(), np.asarray(b).ravel()
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


def relmax(a, b):
    a, b = np.asarray(a).ravel(), np.asarray(b).ravel()
    return np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300)


def make(name, N, eps=None, stop=spp.SPP_STOP_REL_JACOBI, tol=None, sigma=2.0, bx=1.0, by=1.0,
         device=True, **opt):
    cfg = si.config(name, N=N, eps=eps)
    x = spp.spp_shishkin_mesh(N, cfg.eps, sigma, bx)
    y = spp.spp_shishkin_mesh(N, cfg.eps, sigma, by)
    c1, c2, r, f = si.sample_2d(cfg, x, y)
    o = spp.spp_default_options(2)
    o.stop = stop
    o.tol = cfg.tol if tol is None else tol
    for k, v in opt.items():
        setattr(o, k, v)
    conv = dev if device else (lambda a: np.ascontiguousarray(a).ravel())
    S = spp.Solver(2, N, cfg.eps, x, y, conv(c1), conv(c2), conv(r), options=o)
    P = oracle.Oracle2D(N, cfg.eps, oracle.mesh(N, cfg.eps, sigma, bx), oracle.mesh(N, cfg.eps, sigma, by),
                        c1, c2, r, mg_red=o.mg_reduction, mg_cap=o.mg_max_cycles, mg_fixed=o.mg_fixed_cycles)
    return cfg, x, y, (c1, c2, r, f), S, P


# ------------------------------------------------------------------ kernels / stages
@pytest.mark.parametrize("name,N,eps", [("cfg4", 64, 1e-8), ("cfg3", 128, 1e-6), ("cfg2", 128, 1e-2)])
def test_matvec(name, N, eps):
    cfg, x, y, (c1, c2, r, f), S, P = make(name, N, eps)
    z = si.random_field(1, (N - 1, N - 1))
    out = torch.zeros((N - 1) ** 2, dtype=torch.float64, device="cuda")
    S.apply_stage("MATVEC", dev(z), out)
    want = P.matvec(z)
    # difference form: each term is rounded once; bound by the magnitude of the terms
    assert relmax(host(out), want) <= 1e-12


@pytest.mark.parametrize("name,N,eps", [("cfg4", 64, 1e-8), ("cfg5", 128, 1e-2), ("cfg3", 256, 1e-6)])
def test_region_stages(name, N, eps):
    cfg, x, y, ins, S, P = make(name, N, eps)
    m = N - 1
    q = si.random_field(2, (m, m))
    # I
    zi = torch.zeros(m * m, dtype=torch.float64, device="cuda")
    S.apply_stage("MII", dev(q), zi)
    want_i = P.stage_I(q)
    assert relmax(host(zi), want_i) <= 1e-12
    # Y then X on top of the oracle's I values
    zy = dev(want_i)
    S.apply_stage("MYY", dev(q), zy)
    want_y = P.stage_Y(q, want_i)
    assert relmax(host(zy), want_y) <= 1e-11
    zx = dev(want_y)
    S.apply_stage("MXX", dev(q), zx)
    want_x = P.stage_X(q, want_y)
    assert relmax(host(zx), want_x) <= 1e-11
    # corner rhs from (q, z)
    bc = torch.zeros((N // 2) ** 2, dtype=torch.float64, device="cuda")
    S.apply_stage("CORNER_RHS", torch.cat([dev(q), dev(want_x)]), bc)
    assert relmax(host(bc), P.corner_rhs(q, want_x)) <= 1e-14


@pytest.mark.parametrize("name,N,eps", [("cfg4", 128, 1e-8), ("exp2d", 64, 1e-5), ("cfg2", 128, 1e-2)])
def test_multigrid_pieces(name, N, eps):
    kw = dict(sigma=2.5, bx=1.99, by=2.99) if name == "exp2d" else {}
    cfg, x, y, ins, S, P = make(name, N, eps, **kw)
    assert S.mg_levels() == P.levels
    for l in range(P.levels):
        nl = P.level_n(l)
        assert S.mg_level_n(l) == nl
        b = si.random_field(10 + l, (nl, nl))
        e0 = si.random_field(20 + l, (nl, nl))
        out = dev(e0)
        S.apply_stage("GS_SWEEP", dev(b), out, level=l)
        assert relmax(host(out), P.gs_sweep(l, b, e0)) <= 1e-12, l
        out = torch.zeros(nl * nl, dtype=torch.float64, device="cuda")
        S.apply_stage("LEVEL_RESIDUAL", torch.cat([dev(b), dev(e0)]), out, level=l)
        assert relmax(host(out), P.level_residual(l, b, e0)) <= 1e-12, l
        out = torch.zeros(nl * nl, dtype=torch.float64, device="cuda")
        S.apply_stage("VCYCLE", dev(b), out, level=l)
        assert relmax(host(out), P.vcycle(l, b)) <= 1e-11, l
        if l + 1 < P.levels:
            nc = P.level_n(l + 1)
            out = torch.zeros(nc * nc, dtype=torch.float64, device="cuda")
            S.apply_stage("RESTRICT", dev(b), out, level=l)
            assert relmax(host(out), P.restrict(l, b)) <= 1e-13, l
            ec = si.random_field(30 + l, (nc, nc))
            out = dev(e0)
            S.apply_stage("PROLONG_ADD", dev(ec), out, level=l)
            assert relmax(host(out), P.prolong_add(l, ec, e0)) <= 1e-14, l


@pytest.mark.parametrize("name,N,eps", [("cfg4", 128, 1e-8), ("cfg5", 256, 1e-2), ("cfg3", 256, 1e-6)])
def test_product_path_hooks(name, N, eps):
    """The hooks that drive exactly the BASELINE-mode kernels and arguments (spp.h): the z-form
    M_II chain of the Jacobi-weighted solve (input D v, reading R11), the post-smoothing with the
    prolongation fused into the sweep's right-hand-side kernel, and the fused residual +
    restriction with the V-cycle's z-form scalings -- each against the oracle's definition."""
    cfg, x, y, ins, S, P = make(name, N, eps)
    m = N - 1
    D = P.coef()["D"]
    q = si.random_field(3, (m, m))
    zi = torch.zeros(m * m, dtype=torch.float64, device="cuda")
    S.apply_stage("MII_JACOBI", dev(q), zi)
    assert relmax(host(zi), P.stage_I(D * q)) <= 1e-12
    for l in range(P.levels - 1):
        nl, nc = P.level_n(l), P.level_n(l + 1)
        b = si.random_field(50 + l, (nl, nl))
        e0 = si.random_field(60 + l, (nl, nl))
        ec = si.random_field(70 + l, (nc, nc))
        out = torch.zeros(nl * nl, dtype=torch.float64, device="cuda")
        S.apply_stage("POST_SMOOTH", torch.cat([dev(b), dev(e0), dev(ec)]), out, level=l)
        assert relmax(host(out), P.gs_sweep(l, b, P.prolong_add(l, ec, e0))) <= 1e-12, l
        out = torch.zeros(nc * nc, dtype=torch.float64, device="cuda")
        S.apply_stage("RESID_RESTRICT", torch.cat([dev(b), dev(e0)]), out, level=l)
        want = P.restrict(l, P.level_residual(l, b, e0)) / P.level_coef(l + 1)["D"]
        assert relmax(host(out), want) <= 1e-12, l
        # the V-cycle's pair: pre-smoothing from zero, then the restriction of its residual
        # (formed on the GPU as aW e_W + aS e_S; the oracle forms b - A_l e)
        out = torch.zeros(nc * nc, dtype=torch.float64, device="cuda")
        S.apply_stage("PRE_RESTRICT", dev(b), out, level=l)
        e1 = P.gs_sweep(l, b, np.zeros((nl, nl)))
        want = P.restrict(l, P.level_residual(l, b, e1)) / P.level_coef(l + 1)["D"]
        assert relmax(host(out), want) <= 1e-12, l


@pytest.mark.parametrize("name,N,eps", [("cfg4", 256, 1e-8), ("exp2d", 128, 1e-4), ("cfg2", 128, 1e-2)])
def test_corner_solve_and_precond(name, N, eps):
    kw = dict(sigma=2.5, bx=1.99, by=2.99) if name == "exp2d" else {}
    cfg, x, y, ins, S, P = make(name, N, eps, **kw)
    n, m = N // 2, N - 1
    b = si.random_field(40, (n, n))
    out = torch.zeros(n * n, dtype=torch.float64, device="cuda")
    cyc = S.apply_stage("CORNER_SOLVE", dev(b), out)
    zc, cyc_o, _ = P.corner_solve(b)
    assert cyc == cyc_o
    assert rel(host(out), zc) <= 1e-11
    q = si.random_field(41, (m, m))
    out = torch.zeros(m * m, dtype=torch.float64, device="cuda")
    cyc = S.apply_stage("PRECOND", dev(q), out)
    want = P.precond(q)
    assert cyc == P.cycle_log()[-1]
    assert rel(host(out), want) <= 1e-11


# ------------------------------------------------------------------ whole solves
def _solve_pair(name, N, eps=None, stop=spp.SPP_STOP_REL_JACOBI, tol=None, device=True, **kw):
    mesh = {k: kw.pop(k) for k in ("sigma", "bx", "by") if k in kw}
    cfg, x, y, (c1, c2, r, f), S, P = make(name, N, eps, stop=stop, tol=tol, device=device, **mesh, **kw)
    weighted = 1 if stop == spp.SPP_STOP_REL_JACOBI else 0
    stop_abs = 1 if stop == spp.SPP_STOP_ABS_L2 else 0
    t = S.opt.tol
    res = S.solve(dev(f) if device else np.ascontiguousarray(f).ravel())
    ores = P.solve(f, weighted=weighted, stop_abs=stop_abs, tol=t, maxit=S.opt.max_iters,
                   fixed_iters=S.opt.fixed_iters)
    u = host(res.u) if device else res.u
    return cfg, x, y, f, res, ores, u


@pytest.mark.parametrize("name,N,eps", [
    ("cfg2", 128, None),          # BASELINE cfg2 at its size (51-52 iterations, eps N = 1.28)
    ("cfg3", 256, None), ("cfg4", 256, 1e-8), ("cfg4", 512, 1e-6),
    ("cfg5", 256, 1e-2), ("cfg5", 512, 1e-4), ("cfg5", 512, 1e-10),
])
def test_fgmres_parity(name, N, eps):
    cfg, x, y, f, res, ores, u = _solve_pair(name, N, eps)
    assert res.status == ores["status"]
    assert abs(res.stats["iters"] - ores["iters"]) <= 1
    assert res.stats["iters"] == ores["iters"], (res.stats["iters"], ores["iters"])
    assert rel(u, ores["u"]) <= 1e-9
    assert res.stats["mg_cycles_total"] == ores["mg_cycles_total"]
    np.testing.assert_allclose(res.hist, ores["hist"], rtol=1e-6, atol=1e-14 * ores["hist"][0])


@pytest.mark.parametrize("N", [128, 256])
def test_paper_mode_table7_on_gpu(N):
    """Paper mode on the GPU path: eq:exponential_MMS, sigma = 5/2, stop ||R||_2 <=
    10 N^{-1} ln N: Table 7 counts and Table 6 errors."""
    from conftest import load_table, rounds_to
    t6, t7 = load_table("table6_exp_errors.txt"), load_table("table7_exp_iters.txt")
    col = {128: 0, 256: 1}[N]
    for eps in sorted(t7):
        cfg, x, y, f, res, ores, u = _solve_pair("exp2d", N, eps, stop=spp.SPP_STOP_ABS_L2,
                                                 sigma=2.5, bx=1.99, by=2.99)
        assert res.stats["iters"] == int(t7[eps][col])
        assert res.stats["mg_cycles_min"] == 5 and res.stats["mg_cycles_max"] == 5
        err = np.max(np.abs(u.reshape(N - 1, N - 1) - si.exact_solution(cfg, x, y)))
        assert rounds_to(err, t6[eps][col])
        # Paper mode minimises the UNWEIGHTED residual, whose rows scale like eps/h^2 (~1e13 at
        # eps = 1e-7): the loosely stopped iterate (||R|| <= 10 ln N / N) amplifies rounding
        # (reading R11).  The bar is 1e-9, or -- where the oracle itself is less stable
        # than that -- 10x the oracle's own response to a 1e-15 relative perturbation of f
        # (measured: the GPU gap tracks it, 6e-9 at N = 256, eps = 1e-7).
        assert rel(u, ores["u"]) <= max(1e-9, 10 * _oracle_sensitivity("exp2d", N, eps, ores["u"]))


def _oracle_sensitivity(name, N, eps, u_ref):
    """Relative change of the oracle's paper-mode iterate when f is perturbed by 1e-15 (relative,
    seeded): the rounding amplification of the unweighted problem, measured on the oracle alone."""
    cfg = si.config(name, N=N, eps=eps)
    x = oracle.mesh(N, cfg.eps, 2.5, 1.99)
    y = oracle.mesh(N, cfg.eps, 2.5, 2.99)
    c1, c2, r, f = si.sample_2d(cfg, x, y)
    fp = f * (1.0 + 1e-15 * si.random_field(99, f.shape))
    P = oracle.Oracle2D(N, cfg.eps, x, y, c1, c2, r)
    res = P.solve(fp, weighted=0, stop_abs=1, tol=cfg.tol)
    P.close()
    return rel(res["u"], u_ref)


def test_paper_mode_sensitivity_is_conditioning():
    """The paper-mode gaps are the problem's conditioning, not an implementation difference: at
    eps = 1e-4 the oracle's response to a 1e-15 perturbation of f is tiny and the GPU matches
    to 1e-12; at eps = 1e-7 both are orders of magnitude larger, and of the same size."""
    out = {}
    for eps in (1e-4, 1e-7):
        cfg, x, y, f, res, ores, u = _solve_pair("exp2d", 256, eps, stop=spp.SPP_STOP_ABS_L2, sigma=2.5, bx=1.99,
                                                 by=2.99)
        out[eps] = (rel(u, ores["u"]), _oracle_sensitivity("exp2d", 256, eps, ores["u"]))
    assert out[1e-4][0] <= 1e-12
    assert out[1e-7][1] > 100 * out[1e-4][1]
    assert out[1e-7][0] <= 10 * out[1e-7][1]


def test_host_and_device_buffers_agree():
    cfg, x, y, f, r1, o1, u1 = _solve_pair("cfg4", 128, 1e-8, device=True)
    cfg, x, y, f, r2, o2, u2 = _solve_pair("cfg4", 128, 1e-8, device=False)
    assert np.array_equal(u1, u2) and r1.stats["iters"] == r2.stats["iters"]


def test_full_size_cfg3():
    """cfg3 (B:9) at its BASELINE size, full parity with the oracle."""
    cfg, x, y, f, res, ores, u = _solve_pair("cfg3", 1024)
    assert res.stats["iters"] == ores["iters"] == 6
    assert rel(u, ores["u"]) <= 1e-9


def test_full_size_cfg4_bench_config():
    """cfg4 (B:10) at the size bench.py times (4096^2, 16.8M unknowns): full parity."""
    cfg, x, y, f, res, ores, u = _solve_pair("cfg4", 4096)
    assert res.stats["iters"] == ores["iters"]
    assert rel(u, ores["u"]) <= 1e-9
    assert res.stats["true_res_jacobi_rel"] <= 1.01 * cfg.tol


# ------------------------------------------------------------------ edge cases
def test_smallest_mesh_and_zero_rhs():
    cfg, x, y, f, res, ores, u = _solve_pair("cfg4", 8, 1e-3)
    assert res.stats["iters"] == ores["iters"] and rel(u, ores["u"]) <= 1e-9
    c = si.config("cfg4", N=16, eps=1e-4)
    x = spp.spp_shishkin_mesh(16, 1e-4)
    c1, c2, r, f = si.sample_2d(c, x, x)
    S = spp.Solver(2, 16, 1e-4, x, x, dev(c1), dev(c2), dev(r))
    out = S.solve(torch.zeros(225, dtype=torch.float64, device="cuda"))
    assert out.stats["iters"] == 0 and not torch.any(out.u != 0)


def test_uniform_mesh_eps_one():
    cfg, x, y, f, res, ores, u = _solve_pair("cfg5", 64, 1.0)
    assert res.stats["iters"] == ores["iters"] and rel(u, ores["u"]) <= 1e-9


def test_fixed_modes_and_cap():
    cfg, x, y, f, res, ores, u = _solve_pair("cfg4", 128, 1e-8, fixed_iters=2, mg_fixed_cycles=2)
    assert res.stats["iters"] == 2 == ores["iters"]
    assert rel(u, ores["u"]) <= 1e-9
    # max_iters cap -> SPP_NOT_CONVERGED with the last iterate
    cfg, x, y, f, res, ores, u = _solve_pair("cfg5", 128, 1e-2, max_iters=3)
    assert res.status == spp.SPP_NOT_CONVERGED and res.stats["iters"] == 3
    assert rel(u, ores["u"]) <= 1e-9


def test_errors():
    x = spp.spp_shishkin_mesh(16, 1e-4)
    ones = np.ones(225)
    with pytest.raises(spp.SppError) as e:
        spp.Solver(2, 16, 1e-4, x, x, -ones, ones, ones)
    assert e.value.code == -3
    bad = x.copy(); bad[3] += 1e-3
    with pytest.raises(spp.SppError) as e:
        spp.Solver(2, 16, 1e-4, bad, x, ones, ones, ones)
    assert e.value.code == -2
    with pytest.raises(spp.SppError) as e:
        spp.Solver(2, 12, 1e-4, spp.spp_shishkin_mesh(12, 1e-4), spp.spp_shishkin_mesh(12, 1e-4),
                   np.ones(121), np.ones(121), np.ones(121))
    assert e.value.code == -1


# ------------------------------------------------------------------ 1D (cfg1 and the paper tables)
def _solve1d(name, N, eps, side, stop, tol):
    cfg = si.config(name, N=N, eps=eps)
    beta = 0.99 if name == "ex1d" else 1.0
    x = spp.spp_shishkin_mesh(N, cfg.eps, 2.0, beta)
    c, r, f = si.sample_1d(cfg, x)
    o = spp.spp_default_options(1)
    o.side, o.stop, o.tol = side, stop, tol
    S = spp.Solver(1, N, cfg.eps, x, None, dev(c), None, dev(r), options=o)
    res = S.solve(dev(f))
    ores = oracle.solve1d(N, cfg.eps, oracle.mesh(N, cfg.eps, 2.0, beta), c, r, f, side=side,
                          weighted=1 if stop == 0 else 0, stop_abs=1 if stop == 2 else 0, tol=tol, maxit=o.max_iters)
    return res, ores


def test_cfg1():
    res, ores = _solve1d("cfg1", 256, 1e-4, 0, spp.SPP_STOP_REL_JACOBI, 1e-10)
    assert res.stats["iters"] == ores["iters"]
    assert rel(host(res.u), ores["u"]) <= 1e-9


def test_table2_on_gpu():
    """P:848-865 on the GPU 1D path (left GMRES, true inf-norm stop, K = 1)."""
    from conftest import load_table
    t2 = load_table("table2_1d_iters.txt")
    for eps, row in t2.items():
        for col, N in enumerate([128, 256, 512, 1024, 2048]):
            if row[col] is None:
                continue
            res, ores = _solve1d("ex1d", N, eps, spp.SPP_LEFT, spp.SPP_STOP_ABS_MAX, np.log(N) / N)
            assert res.stats["iters"] == int(row[col]) == ores["iters"], (eps, N)
            assert rel(host(res.u), ores["u"]) <= 1e-9


# ------------------------------------------------------------------ execution-path equivalence
def _with_env(var, fn):
    import os
    old = os.environ.get(var)
    os.environ[var] = "1"
    try:
        return fn()
    finally:
        if old is None:
            del os.environ[var]
        else:
            os.environ[var] = old


@pytest.mark.parametrize("name,N,eps,opt", [("cfg4", 512, 1e-8, {}), ("cfg5", 256, 1e-2, {}),
                                           ("cfg4", 256, 1e-8, {"mg_max_cycles": 2})])
def test_corner_graph_matches_host_loop(name, N, eps, opt):
    """The corner solve as a CUDA graph with a device-side while loop (DESIGN.md "The corner
    solve as a CUDA graph") makes the same per-cycle decisions as the host-driven loop: same
    cycle counts, cap hits and iterates, bit for bit; and both match the oracle."""
    cfg, x, y, f, r_graph, ores, u_graph = _solve_pair(name, N, eps, **opt)
    _, _, _, _, r_host, _, u_host = _with_env("SPP_NO_GRAPH", lambda: _solve_pair(name, N, eps, **opt))
    for k in ("iters", "mg_cycles_total", "mg_cycles_min", "mg_cycles_max", "mg_cap_hits"):
        assert r_graph.stats[k] == r_host.stats[k], k
    assert np.array_equal(u_graph, u_host)
    assert r_graph.stats["mg_cycles_total"] == ores["mg_cycles_total"]
    assert rel(u_graph, ores["u"]) <= 1e-9
    if opt.get("mg_max_cycles"):
        assert r_graph.stats["mg_cap_hits"] == r_graph.stats["iters"] > 0


@pytest.mark.parametrize("name,N,eps,opt", [("cfg2", 128, None, {}), ("cfg4", 256, 1e-8, {"fixed_iters": 3}),
                                           ("cfg5", 256, 1e-4, {"max_iters": 5, "tol": 1e-15}),
                                           ("cfg4", 256, 1e-8, {"mg_fixed_cycles": 2})])
def test_iteration_graphs_match_host_loop(name, N, eps, opt):
    """FGMRES iterations as CUDA graphs (capi.cu "iteration graphs": the Givens update and stop
    test on the device, the corner loop a nested while node, batches of speculative iterations
    behind a device-side gate) against the host-driven loop: the same statistics, residual
    history and iterate, bit for bit; repeated solves on one context (batch sizes from the previous
    solve, graphs reused) too."""
    cfg = si.config(name, N=N, eps=eps)
    x = spp.spp_shishkin_mesh(N, cfg.eps, cfg.sigma, cfg.beta_x)
    y = spp.spp_shishkin_mesh(N, cfg.eps, cfg.sigma, cfg.beta_y)
    c1, c2, r, f = si.sample_2d(cfg, x, y)

    def run():
        o = spp.spp_default_options(2)
        o.tol = cfg.tol
        for k, v in opt.items():
            setattr(o, k, v)
        S = spp.Solver(2, N, cfg.eps, x, y, dev(c1), dev(c2), dev(r), options=o)
        out = []
        for k in range(3):                      # the same rhs, a scaled one, a perturbed one
            fk = f * (1.0 + k) + (k == 2) * si.random_field(500, f.shape)
            res = S.solve(dev(fk))
            out.append((res.status, dict(res.stats), np.array(res.hist), host(res.u)))
        S.close()
        return out

    g = run()
    h = _with_env("SPP_NO_GRAPH", run)
    for (sg, stg, hg, ug), (sh, sth, hh, uh) in zip(g, h):
        assert sg == sh
        for k in ("iters", "converged", "mg_cycles_total", "mg_cycles_min", "mg_cycles_max", "mg_cap_hits",
                  "res_final"):
            assert stg[k] == sth[k], (k, stg[k], sth[k])
        assert np.array_equal(hg, hh)
        assert np.array_equal(ug, uh)
    if "max_iters" in opt:
        assert g[0][1]["iters"] == opt["max_iters"] and not g[0][1]["converged"]


def test_iteration_graphs_cap_failure():
    """mg_strict: a corner cycle-cap hit inside the graphs fails the solve with SPP_E_MG_CAP."""
    cfg = si.config("cfg4", N=256, eps=1e-8)
    x = spp.spp_shishkin_mesh(256, cfg.eps)
    c1, c2, r, f = si.sample_2d(cfg, x, x)
    o = spp.spp_default_options(2)
    o.mg_max_cycles, o.mg_strict = 1, 1
    S = spp.Solver(2, 256, cfg.eps, x, x, dev(c1), dev(c2), dev(r), options=o)
    with pytest.raises(spp.SppError) as ei:
        S.solve(dev(f))
    assert ei.value.code == -5                  # SPP_E_MG_CAP


@pytest.mark.parametrize("name,N,eps", [("cfg3", 1024, None), ("cfg4", 512, 1e-8)])
def test_tma_line_kernel_matches_lsu_kernel(name, N, eps):
    """The TMA-staged line-chain kernel (k_lines_tma, line length a multiple of 128) computes the
    same arithmetic in the same order as the LSU-loaded one: identical results."""
    cfg, x, y, f, r_tma, ores, u_tma = _solve_pair(name, N, eps)
    _, _, _, _, r_lsu, _, u_lsu = _with_env("SPP_NO_LINES_TMA", lambda: _solve_pair(name, N, eps))
    assert r_tma.stats["iters"] == r_lsu.stats["iters"]
    assert np.array_equal(u_tma, u_lsu)
    assert rel(u_tma, ores["u"]) <= 1e-9


@pytest.mark.parametrize("eps", [1e-6, 1e-10])
def test_cfg5_at_2048(eps):
    """cfg5's data (B:11: c = (1,2), r = 1, seeded random f) at N = 2048 (4.2M unknowns): the
    tiled corner levels, the TMA line kernel (lines of 1024) and the 2-warp M_II chain at a size
    between the proxies and the bench, against the oracle."""
    cfg, x, y, f, res, ores, u = _solve_pair("cfg5", 2048, eps)
    assert res.stats["iters"] == ores["iters"]
    assert res.stats["mg_cycles_total"] == ores["mg_cycles_total"]
    assert rel(u, ores["u"]) <= 1e-9


def test_full_size_cfg5_eps_1e10():
    """cfg5 (B:11) at its BASELINE size, 8192^2 (67M unknowns), eps = 1e-10: full parity with the
    oracle (the largest single-GPU configuration; 3 iterations)."""
    cfg, x, y, f, res, ores, u = _solve_pair("cfg5", 8192, 1e-10)
    assert res.stats["iters"] == ores["iters"]
    assert res.stats["mg_cycles_total"] == ores["mg_cycles_total"]
    assert rel(u, ores["u"]) <= 1e-9


@pytest.mark.parametrize("name,N,eps", [("cfg4", 512, 1e-8), ("cfg5", 256, 1e-2)])
def test_scan_line_factorisation_matches_sequential(name, N, eps):
    """The block-scan Thomas factorisation (2x2 matrix prefix products) and the sequential
    per-line sweep give the same preconditioner up to rounding: same iterations, solutions within
    the parity bar of each other and of the oracle."""
    cfg, x, y, f, r_scan, ores, u_scan = _solve_pair(name, N, eps)
    _, _, _, _, r_seq, _, u_seq = _with_env("SPP_SEQ_LINE_FACTOR", lambda: _solve_pair(name, N, eps))
    assert r_scan.stats["iters"] == r_seq.stats["iters"] == ores["iters"]
    assert rel(u_scan, u_seq) <= 1e-12
    assert rel(u_scan, ores["u"]) <= 1e-9


@pytest.mark.parametrize("N", [512, 1024, 2048])
def test_paper_tables_6_7_large_N_on_gpu(N):
    """Paper mode at the larger sizes of Tables 6/7, GPU only, pinned to the
    printed numbers: FGMRES counts exactly (Table 7) and the max-norm error to 4 digits
    (Table 6), every apply taking the paper's 5 corner cycles."""
    from conftest import load_table, rounds_to
    t6, t7 = load_table("table6_exp_errors.txt"), load_table("table7_exp_iters.txt")
    col = {128: 0, 256: 1, 512: 2, 1024: 3, 2048: 4}[N]
    for eps in sorted(t7):
        cfg, x, y, (c1, c2, r, f), S, P = make("exp2d", N, eps, stop=spp.SPP_STOP_ABS_L2, sigma=2.5,
                                                bx=1.99, by=2.99)
        P.close()
        res = S.solve(dev(f))
        u = host(res.u)
        assert res.stats["iters"] == int(t7[eps][col]), (N, eps, res.stats["iters"])
        assert res.stats["mg_cycles_min"] == 5 and res.stats["mg_cycles_max"] == 5
        err = np.max(np.abs(u.reshape(N - 1, N - 1) - si.exact_solution(cfg, x, y)))
        assert rounds_to(err, t6[eps][col]), (N, eps, err)

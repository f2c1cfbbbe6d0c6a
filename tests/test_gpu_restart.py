"""FGMRES(m) on the GPU (spp_options.restart > 0, reading R23) against the oracle's
restarted FGMRES (tests/test_oracle_restart.py pins it to the definition of a GMRES(m) cycle):
identical iteration and corner-cycle counts, solutions within the 1e-9 parity bar."""
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


def _pair(name, N, eps, restart, **opt):
    cfg = si.config(name, N=N, eps=eps)
    x = spp.spp_shishkin_mesh(N, cfg.eps, cfg.sigma, cfg.beta_x)
    y = spp.spp_shishkin_mesh(N, cfg.eps, cfg.sigma, cfg.beta_y)
    c1, c2, r, f = si.sample_2d(cfg, x, y)
    o = spp.spp_default_options(2)
    o.tol = cfg.tol
    o.restart = restart
    for k, v in opt.items():
        setattr(o, k, v)
    S = spp.Solver(2, N, cfg.eps, x, y, dev(c1), dev(c2), dev(r), options=o)
    P = oracle.Oracle2D(N, cfg.eps, oracle.mesh(N, cfg.eps, cfg.sigma, cfg.beta_x),
                        oracle.mesh(N, cfg.eps, cfg.sigma, cfg.beta_y), c1, c2, r)
    return cfg, f, S, P, o


@pytest.mark.parametrize("name,N,eps,m", [("cfg5", 256, 1e-2, 10), ("cfg5", 512, 1e-4, 4), ("cfg4", 512, 1e-6, 2),
                                          ("cfg2", 128, 1e-2, 8)])
def test_restarted_solve_matches_oracle(name, N, eps, m):
    cfg, f, S, P, o = _pair(name, N, eps, m, max_iters=400)
    res = S.solve(dev(f), hist_cap=512)
    ores = P.solve(f, weighted=1, stop_abs=0, tol=o.tol, maxit=o.max_iters, restart=m)
    assert res.stats["iters"] == ores["iters"] and res.stats["iters"] > m    # at least one restart
    assert res.stats["mg_cycles_total"] == ores["mg_cycles_total"]
    assert res.status == spp.SPP_OK and ores["converged"]
    assert rel(res.u.cpu().numpy(), ores["u"]) <= 1e-9
    h, oh = res.hist, ores["hist"]
    assert np.max(np.abs(h - oh) / oh) <= 1e-6                                # residual history
    # the host-driven loop (profiling) runs the same kernels: bit for bit the graph path
    S.profile_enable(1)
    res2 = S.solve(dev(f), hist_cap=512)
    assert torch.equal(res2.u, res.u) and np.array_equal(res2.hist, res.hist)


def test_restart_at_or_above_the_count_is_the_unrestarted_solve():
    cfg, f, S, P, o = _pair("cfg4", 512, 1e-8, 0)
    a = S.solve(dev(f))
    for m in (a.stats["iters"], 50):
        _, _, S2, _, _ = _pair("cfg4", 512, 1e-8, m)
        b = S2.solve(dev(f))
        assert torch.equal(a.u, b.u) and np.array_equal(a.hist, b.hist)


def test_restart_with_the_iteration_cap():
    # 25 steps in cycles of 10: SPP_NOT_CONVERGED with the iterate after the partial third cycle
    cfg, f, S, P, o = _pair("cfg5", 256, 1e-2, 10, max_iters=25)
    res = S.solve(dev(f), hist_cap=64)
    ores = P.solve(f, weighted=1, stop_abs=0, tol=o.tol, maxit=25, restart=10)
    assert res.status == spp.SPP_NOT_CONVERGED and res.stats["iters"] == 25 == ores["iters"]
    assert not ores["converged"]
    assert rel(res.u.cpu().numpy(), ores["u"]) <= 1e-9

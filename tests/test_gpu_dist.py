"""Row strips on one GPU: P strips with the loopback transport run
the distributed algorithm -- every exchange step, halo, relay and all-gather of the multi-GPU
solve -- and must reproduce the single-GPU solve: identical FGMRES iteration and corner cycle
counts, solutions within 1e-12 relative l2 of the one-strip solve (the strips change only the
summation order of the dot products and the certified-halo truncation, both below fp64
rounding), and within the 1e-9 parity bar of the oracle."""
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


def _inputs(name, N, eps, **opt):
    cfg = si.config(name, N=N, eps=eps)
    x = spp.spp_shishkin_mesh(N, cfg.eps, cfg.sigma, cfg.beta_x)
    y = spp.spp_shishkin_mesh(N, cfg.eps, cfg.sigma, cfg.beta_y)
    c1, c2, r, f = si.sample_2d(cfg, x, y)
    o = spp.spp_default_options(2)
    o.tol = cfg.tol
    for k, v in opt.items():
        setattr(o, k, v)
    return cfg, x, y, (c1, c2, r, f), o


def _solve(cfg, x, y, data, o, strips):
    c1, c2, r, f = data
    S = spp.Solver(2, cfg.N, cfg.eps, x, y, dev(c1), dev(c2), dev(r), options=o, strips=strips)
    res = S.solve(dev(f))
    info = S.dist_info()
    u = res.u.cpu().numpy()
    S.close()
    return res, u, info


@pytest.mark.parametrize("name,N,eps,P", [
    ("cfg4", 128, 1e-8, 2), ("cfg4", 256, 1e-8, 3), ("cfg4", 256, 1e-8, 4), ("cfg4", 512, 1e-8, 8),
    ("cfg5", 256, 1e-6, 2), ("cfg3", 512, 1e-6, 4), ("cfg2", 128, 1e-2, 2), ("cfg5", 512, 1e-4, 5),
    ("cfg4", 512, 1e-8, 6), ("cfg4", 256, 1e-8, 7),
])
def test_strips_match_one_gpu_and_oracle(name, N, eps, P):
    cfg, x, y, data, o = _inputs(name, N, eps)
    r1, u1, _ = _solve(cfg, x, y, data, o, 1)
    rP, uP, info = _solve(cfg, x, y, data, o, P)
    assert info["nranks"] == P and info["strip_levels"] >= 1 and info["xfers"] > 0
    assert rP.stats["iters"] == r1.stats["iters"], (rP.stats["iters"], r1.stats["iters"])
    assert rP.stats["mg_cycles_total"] == r1.stats["mg_cycles_total"]
    assert rel(uP, u1) <= 1e-12, rel(uP, u1)
    assert np.allclose(rP.hist, r1.hist, rtol=1e-9, atol=0)
    Po = oracle.Oracle2D(N, cfg.eps, oracle.mesh(N, cfg.eps), oracle.mesh(N, cfg.eps), *data[:3])
    ores = Po.solve(data[3], weighted=1, tol=cfg.tol)
    Po.close()
    assert rP.stats["iters"] == ores["iters"]
    assert rel(uP, ores["u"]) <= 1e-9


@pytest.mark.parametrize("dl", [1, 2, 3])
def test_strip_levels_and_host_buffers(dl, monkeypatch):
    """Every number of corner levels smoothed on the strips gives the same solve; host (numpy)
    buffers through the strips equal device ones."""
    monkeypatch.setenv("SPP_TUNE", f"dist_levels={dl}")
    cfg, x, y, data, o = _inputs("cfg4", 512, 1e-8)
    r1, u1, _ = _solve(cfg, x, y, data, o, 1)
    rP, uP, info = _solve(cfg, x, y, data, o, 4)
    assert info["strip_levels"] == dl
    assert rP.stats["iters"] == r1.stats["iters"] and rP.stats["mg_cycles_total"] == r1.stats["mg_cycles_total"]
    assert rel(uP, u1) <= 1e-12
    c1, c2, r, f = data
    S = spp.Solver(2, cfg.N, cfg.eps, x, y, *(np.ascontiguousarray(a).ravel() for a in (c1, c2, r)), options=o, strips=4)
    rh = S.solve(np.ascontiguousarray(f).ravel())
    assert rh.stats["iters"] == rP.stats["iters"]
    assert np.array_equal(rh.u, uP)


def test_strips_fixed_modes_and_true_residual():
    """Parity modes (fixed iterations / fixed cycles) and the true-residual statistics on strips."""
    cfg, x, y, data, o = _inputs("cfg4", 256, 1e-8, fixed_iters=2, mg_fixed_cycles=3)
    r1, u1, _ = _solve(cfg, x, y, data, o, 1)
    rP, uP, _ = _solve(cfg, x, y, data, o, 3)
    assert rP.stats["iters"] == r1.stats["iters"] == 2
    assert rP.stats["mg_cycles_total"] == r1.stats["mg_cycles_total"] == 6
    assert rel(uP, u1) <= 1e-12
    for k in ("true_res_l2_rel", "true_res_jacobi_rel"):
        assert abs(rP.stats[k] - r1.stats[k]) <= 1e-9 * max(r1.stats[k], 1e-300) + 1e-14


@pytest.mark.parametrize("P", [2, 4, 8])
def test_full_size_cfg4_on_strips(P):
    """cfg4 at its BASELINE size (4096^2, 16.8M unknowns, B:10), the configuration north_star
    shards across 1/2/4/8 GPUs: P strips match the single-GPU solve to 1e-12 with identical
    iteration and corner-cycle counts."""
    cfg, x, y, data, o = _inputs("cfg4", 4096, 1e-8)
    r1, u1, _ = _solve(cfg, x, y, data, o, 1)
    rP, uP, info = _solve(cfg, x, y, data, o, P)
    assert rP.stats["iters"] == r1.stats["iters"]
    assert rP.stats["mg_cycles_total"] == r1.stats["mg_cycles_total"]
    assert rel(uP, u1) <= 1e-12, rel(uP, u1)


def test_strip_errors():
    cfg, x, y, (c1, c2, r, f), o = _inputs("cfg4", 16, 1e-8)
    with pytest.raises(spp.SppError):                       # 16 strips cannot fit N = 16
        spp.Solver(2, 16, cfg.eps, x, y, dev(c1), dev(c2), dev(r), options=o, strips=16)
    S = spp.Solver(2, 16, cfg.eps, x, y, dev(c1), dev(c2), dev(r), options=o, strips=2)
    with pytest.raises(spp.SppError) as ei:                 # test hooks are single-GPU only
        S.apply_stage("MATVEC", dev(f), torch.zeros(15 * 15, dtype=torch.float64, device="cuda"))
    assert ei.value.code == -9
    ff = np.ascontiguousarray(f).ravel().copy()
    ff[3] = np.nan
    with pytest.raises(spp.SppError) as ei:
        S.solve(dev(ff))
    assert ei.value.code == -10

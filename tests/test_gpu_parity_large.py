"""GPU-vs-oracle parity at the configurations whose oracle runs take minutes (VERDICT r1
"parity gaps"): cfg5 (B:11) at its BASELINE size 8192^2 for eps = 1e-8 (5 iterations) and
eps = 1e-6 (23 iterations, 25 GB of oracle Krylov vectors), and the two cells that do not
converge in 100 iterations (eps = 1e-2, 1e-4; a common cap on both sides) at
N = 2048.  The four oracle solves start together in worker threads when the module is first
used (the oracle's C code runs without the GIL), so the wall time is the slowest one (~3.5 min
on the box's host cores), not their sum.  Bars as test_gpu_parity: identical iteration and
corner-cycle counts, <= 1e-9 relative l2."""
import concurrent.futures as cf

import numpy as np
import pytest

import oracle
import spp_inputs as si

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2108_13468_b200 as spp  # noqa: E402

CASES = {"8192-1e-8": (8192, 1e-8, 200), "8192-1e-6": (8192, 1e-6, 200),
         "2048-1e-2": (2048, 1e-2, 100), "2048-1e-4": (2048, 1e-4, 100)}
_POOL = None
_JOBS = {}


def _inputs(N, eps):
    cfg = si.config("cfg5", N=N, eps=eps)
    x = oracle.mesh(N, cfg.eps)
    c1, c2, r, f = si.sample_2d(cfg, x, x)
    return cfg, x, (c1, c2, r, f)


def _oracle_job(N, eps, maxit):
    cfg, x, (c1, c2, r, f) = _inputs(N, eps)
    P = oracle.Oracle2D(N, cfg.eps, x, x, c1, c2, r)
    res = P.solve(f, weighted=1, tol=cfg.tol, maxit=maxit)
    P.close()
    return {k: res[k] for k in ("u", "iters", "mg_cycles_total", "converged", "hist")}


def _oracle(key):
    global _POOL
    if _POOL is None:
        _POOL = cf.ThreadPoolExecutor(max_workers=len(CASES))
        for k, args in CASES.items():
            _JOBS[k] = _POOL.submit(_oracle_job, *args)
    return _JOBS[key].result()


@pytest.mark.parametrize("key", list(CASES))
def test_cfg5_large_parity(key):
    _oracle(key)                                   # starts all four oracle solves on first use
    N, eps, maxit = CASES[key]
    cfg, x, (c1, c2, r, f) = _inputs(N, eps)
    xs = spp.spp_shishkin_mesh(N, cfg.eps)
    assert np.array_equal(xs, x)
    o = spp.spp_default_options(2)
    o.tol, o.max_iters = cfg.tol, maxit
    d = lambda a: torch.from_numpy(np.ascontiguousarray(a).ravel()).cuda()
    S = spp.Solver(2, N, cfg.eps, xs, xs, d(c1), d(c2), d(r), options=o)
    res = S.solve(d(f))
    u = res.u.cpu().numpy()
    S.close()
    ores = _oracle(key)
    assert res.stats["iters"] == ores["iters"], (res.stats["iters"], ores["iters"])
    assert res.stats["mg_cycles_total"] == ores["mg_cycles_total"]
    assert bool(res.stats["converged"]) == ores["converged"]
    assert np.linalg.norm(u - ores["u"].ravel()) <= 1e-9 * np.linalg.norm(ores["u"])
    np.testing.assert_allclose(res.hist, ores["hist"], rtol=1e-6, atol=1e-14 * ores["hist"][0])

"""Measure parity margins and oracle costs on the GPU box (diagnostics for DESIGN.md / tests):
paper-mode GPU-vs-oracle gaps, and the oracle's wall time for the large parity cases."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import oracle  # noqa: E402
import paper_2108_13468_b200 as spp  # noqa: E402
import spp_inputs as si  # noqa: E402


def run(name, N, eps, stop=spp.SPP_STOP_REL_JACOBI, sigma=2.0, bx=1.0, by=1.0, maxit=200, tol=None):
    cfg = si.config(name, N=N, eps=eps)
    x = spp.spp_shishkin_mesh(N, cfg.eps, sigma, bx)
    y = spp.spp_shishkin_mesh(N, cfg.eps, sigma, by)
    c1, c2, r, f = si.sample_2d(cfg, x, y)
    o = spp.spp_default_options(2)
    o.stop, o.tol, o.max_iters = stop, cfg.tol if tol is None else tol, maxit
    d = lambda a: torch.from_numpy(np.ascontiguousarray(a).ravel()).cuda()
    t0 = time.time()
    S = spp.Solver(2, N, cfg.eps, x, y, d(c1), d(c2), d(r), options=o)
    res = S.solve(d(f))
    tg = time.time() - t0
    u = res.u.cpu().numpy()
    S.close()
    t0 = time.time()
    P = oracle.Oracle2D(N, cfg.eps, oracle.mesh(N, cfg.eps, sigma, bx), oracle.mesh(N, cfg.eps, sigma, by), c1, c2, r)
    ores = P.solve(f, weighted=1 if stop == spp.SPP_STOP_REL_JACOBI else 0,
                   stop_abs=1 if stop == spp.SPP_STOP_ABS_L2 else 0, tol=o.tol, maxit=maxit)
    P.close()
    to = time.time() - t0
    e = np.linalg.norm(u - ores["u"].ravel()) / np.linalg.norm(ores["u"])
    print(f"{name} N={N} eps={eps:g}: gpu iters {res.stats['iters']} cyc {res.stats['mg_cycles_total']} | oracle "
          f"{ores['iters']} cyc {ores['mg_cycles_total']} | rel {e:.3e} | gpu {tg:.1f}s oracle {to:.1f}s", flush=True)


which = sys.argv[1] if len(sys.argv) > 1 else "paper"
if which == "paper":
    for N in (128, 256, 512):
        for eps in (1e-4, 1e-5, 1e-6, 1e-7):
            run("exp2d", N, eps, stop=spp.SPP_STOP_ABS_L2, sigma=2.5, bx=1.99, by=2.99, tol=10 * np.log(N) / N)
elif which == "cap":
    for eps in (1e-2, 1e-4):
        run("cfg5", 2048, eps, maxit=100)
elif which == "big":
    for eps in (1e-8, 1e-6):
        run("cfg5", 8192, eps)

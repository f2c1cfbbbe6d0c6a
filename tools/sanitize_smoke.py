"""Small solves for compute-sanitizer (memcheck): 2D N=64 (cfg4 data, tiled + chained sweeps,
lines, corner graph) and 1D; exits non-zero on a CUDA error."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2108_13468_b200 as spp  # noqa: E402
import spp_inputs as si  # noqa: E402

for name, N, eps in [("cfg4", 64, 1e-8), ("cfg5", 128, 1e-2)]:
    cfg = si.config(name, N=N, eps=eps)
    x = spp.spp_shishkin_mesh(N, cfg.eps, cfg.sigma, cfg.beta_x)
    y = spp.spp_shishkin_mesh(N, cfg.eps, cfg.sigma, cfg.beta_y)
    c1, c2, r, f = si.sample_2d(cfg, x, y)
    d = [torch.from_numpy(np.ascontiguousarray(a).ravel()).cuda() for a in (c1, c2, r, f)]
    S = spp.Solver(2, N, cfg.eps, x, y, d[0], d[1], d[2])
    res = S.solve(d[3])
    res = S.solve(d[3])   # second solve replays the corner graph
    torch.cuda.synchronize()
    print(name, N, "iters", res.stats["iters"], "true res", res.stats["true_res_jacobi_rel"])
print("sanitize smoke done")

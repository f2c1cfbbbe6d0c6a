"""Paper-mode timings on the GPU next to the paper's Table 7 CPU times.

Exponential-layer MMS, sigma = 5/2, C = (1.99, 2.99), stop ||R||_2 <= 10 N^-1 ln N
(P:1313).  Time = spp_setup + spp_solve (device buffers, CUDA events around both, after one
warm-up solve of the same problem), i.e. the paper's "all costs for the setup and preconditioned
FGMRES iterations".  The paper's hardware is its own CPU."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2108_13468_b200 as spp  # noqa: E402
import spp_inputs as si  # noqa: E402

PAPER = {  # eps: [(seconds, iterations) for N = 2^7 .. 2^11]
    1e-4: [(0.010, 3), (0.041, 4), (0.266, 6), (2.656, 14), (37.690, 40)],
    1e-5: [(0.010, 4), (0.041, 4), (0.178, 4), (1.103, 6), (7.625, 10)],
    1e-6: [(0.010, 4), (0.041, 4), (0.221, 5), (0.921, 5), (3.771, 5)],
    1e-7: [(0.010, 4), (0.051, 5), (0.221, 5), (0.923, 5), (4.519, 6)],
}


def main():
    dev = torch.device("cuda", 0)
    print(f"# GPU: {torch.cuda.get_device_name(0)}; paper: its own CPU (Table 7)")
    print("# eps      N   iters(paper) iters(gpu)   paper_s     gpu_ms   speedup")
    for eps in sorted(PAPER, reverse=True):
        for col, N in enumerate([128, 256, 512, 1024, 2048]):
            cfg = si.config("exp2d", N=N, eps=eps)
            x = spp.spp_shishkin_mesh(N, eps, 2.5, 1.99)
            y = spp.spp_shishkin_mesh(N, eps, 2.5, 2.99)
            c1, c2, r, f = si.sample_2d(cfg, x, y)
            d = [torch.from_numpy(np.ascontiguousarray(a).ravel()).to(dev) for a in (c1, c2, r, f)]
            o = spp.spp_default_options(2)
            o.stop = spp.SPP_STOP_ABS_L2
            o.tol = cfg.tol
            S = spp.Solver(2, N, eps, x, y, d[0], d[1], d[2], options=o)
            S.setup(d[0], d[1], d[2])
            S.solve(d[3])
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            S.setup(d[0], d[1], d[2])
            res = S.solve(d[3])
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1)
            ps, pit = PAPER[eps][col]
            print(f"{eps:7.0e} {N:5d} {pit:8d} {res.stats['iters']:10d} {ps:10.3f} {ms:10.2f} {ps * 1e3 / ms:9.0f}x")


if __name__ == "__main__":
    main()

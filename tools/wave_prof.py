"""Per-warp timing of one k_wave launch (SPP_WAVE_PROF build): one cfg4 solve, the dump of the
SPP_WAVE_PROF_HIT-th launch over a level of SPP_WAVE_PROF_N columns goes to stderr."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2108_13468_b200 as spp  # noqa: E402
import spp_inputs as si  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
cfg = si.config("cfg4", N=N)
x = spp.spp_shishkin_mesh(N, cfg.eps)
c1, c2, r, f = si.sample_2d(cfg, x, x)
d = lambda a: torch.from_numpy(np.ascontiguousarray(a).ravel()).cuda()
o = spp.spp_default_options(2)
S = spp.Solver(2, N, cfg.eps, x, x, d(c1), d(c2), d(r), options=o)
S.profile_enable(1)          # host-driven corner loop (the dump syncs the stream)
res = S.solve(d(f))
print("iters", res.stats["iters"])

"""Run the GS_SWEEP stage hook level by level with synchronous error reporting."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["SPP_DEBUG_SYNC"] = "1"
import numpy as np, torch
import paper_2108_13468_b200 as spp, spp_inputs as si
N, eps = int(sys.argv[1]) if len(sys.argv) > 1 else 128, 1e-8
cfg = si.config("cfg4", N=N, eps=eps)
x = spp.spp_shishkin_mesh(N, eps)
c1, c2, r, f = si.sample_2d(cfg, x, x)
d = lambda a: torch.from_numpy(np.ascontiguousarray(a).ravel()).cuda()
S = spp.Solver(2, N, eps, x, x, d(c1), d(c2), d(r))
for l in range(S.mg_levels()):
    nl = S.mg_level_n(l)
    print("level", l, nl, flush=True)
    b = d(si.random_field(1, (nl, nl))); out = d(si.random_field(2, (nl, nl)))
    try:
        S.apply_stage("GS_SWEEP", b, out, level=l)
    except Exception as e:
        print("FAILED", e, flush=True); break

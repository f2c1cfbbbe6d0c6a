"""Worker of tests/test_gpu_dist_proc.py::test_lost_peer_is_an_error_not_a_hang: two ranks build
their strips (collective), then rank 1 leaves without solving.  Rank 0's solve must come back
with SPP_E_NCCL (from the transport's / dist_wait's timeout), not hang."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2108_13468_b200 as spp  # noqa: E402
import spp_inputs as si  # noqa: E402

N = 128
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(0)
dist.init_process_group("gloo")
cfg = si.config("cfg4", N=N)
x = spp.spp_shishkin_mesh(N, cfg.eps)
c1, c2, r, f = si.sample_2d(cfg, x, x)
J = spp.spp_strip_partition(N, world)
j0, j1 = int(J[rank]), int(J[rank + 1])
rows = slice(j0 - 1, j1 - 1)
d = [torch.from_numpy(np.ascontiguousarray(a[rows]).ravel()).cuda() for a in (c1, c2, r, f)]
obj = [spp.nccl_unique_id() if rank == 0 else None]
dist.broadcast_object_list(obj, src=0)
comm = spp.nccl_comm_create(obj[0], world, rank)
o = spp.spp_default_options(2)
o.tol = cfg.tol
S = spp.DistSolver(N, cfg.eps, x, x, d[0], d[1], d[2], j0, j1, comm, rank, world, options=o)
dist.barrier()
if rank == 0:
    try:
        S.solve(d[3])
        print("UNEXPECTED: solve returned")
    except spp.SppError as e:
        print(f"rank 0: SppError code {e.code}: {e}")
        print("LOST PEER DETECTED" if e.code == spp.SPP_E_NCCL else "WRONG CODE")
dist.destroy_process_group()
os._exit(0)          # no collective teardown: the peer is gone

"""Functional check of the one-strip-per-process path (spp_create_dist) when only ONE GPU is
available: every rank of a torchrun job uses cuda:0 (NOT a measurement: the ranks share one
device).  Each rank solves its strip of the problem and rank 0 compares the gathered solution
with the single-GPU solve (same iterations and corner cycles, <= 1e-12 relative l2).

The real NCCL refuses two ranks on one device ("invalid usage"), so on a one-GPU box point
SPP_NCCL_LIB at tests/mock_nccl/libmock_nccl.so (tests/test_gpu_dist_proc.py does); on a
multi-GPU node change set_device(0) to LOCAL_RANK and it runs over the real NCCL.

    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 tools/nccl_strips_check.py [N] [cfg]
"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2108_13468_b200 as spp  # noqa: E402
import spp_inputs as si  # noqa: E402


def main():
    N = int(sys.argv[1]) if len(sys.argv) > 1 else 256
    name = sys.argv[2] if len(sys.argv) > 2 else "cfg4"
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    ngpu = torch.cuda.device_count()
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")) if ngpu >= world else 0)
    dist.init_process_group("gloo")
    cfg = si.config(name, N=N)
    x = spp.spp_shishkin_mesh(N, cfg.eps, cfg.sigma, cfg.beta_x)
    y = spp.spp_shishkin_mesh(N, cfg.eps, cfg.sigma, cfg.beta_y)
    c1, c2, r, f = si.sample_2d(cfg, x, y)
    J = spp.spp_strip_partition(N, world)
    j0, j1 = int(J[rank]), int(J[rank + 1])
    rows = slice(j0 - 1, j1 - 1)
    d = [torch.from_numpy(np.ascontiguousarray(a[rows]).ravel()).cuda() for a in (c1, c2, r, f)]
    obj = [spp.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    comm = spp.nccl_comm_create(obj[0], world, rank)
    o = spp.spp_default_options(2)
    o.stop = spp.SPP_STOP_REL_JACOBI if cfg.weighted else (spp.SPP_STOP_ABS_L2 if cfg.stop_abs else spp.SPP_STOP_REL_L2)
    o.tol = cfg.tol
    S = spp.DistSolver(N, cfg.eps, x, y, d[0], d[1], d[2], j0, j1, comm, rank, world, options=o)
    res = S.solve(d[3])
    parts = [None] * world
    dist.all_gather_object(parts, (res.u.cpu().numpy(), res.stats))
    if rank == 0:
        u = np.concatenate([p[0] for p in parts])
        S1 = spp.Solver(2, N, cfg.eps, x, y, *(torch.from_numpy(np.ascontiguousarray(a).ravel()).cuda()
                                                for a in (c1, c2, r)), options=o)
        r1 = S1.solve(torch.from_numpy(np.ascontiguousarray(f).ravel()).cuda())
        u1 = r1.u.cpu().numpy()
        e = np.linalg.norm(u - u1) / np.linalg.norm(u1)
        ok = (res.stats["iters"] == r1.stats["iters"] and res.stats["mg_cycles_total"] == r1.stats["mg_cycles_total"]
              and e <= 1e-12)
        print(f"nccl strips {name} N={N} P={world}: iters {res.stats['iters']} vs {r1.stats['iters']}, cycles "
              f"{res.stats['mg_cycles_total']} vs {r1.stats['mg_cycles_total']}, rel {e:.3e} -> {'OK' if ok else 'FAIL'}")
        print(S.dist_info())
    S.close()
    spp.nccl_comm_destroy(comm)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()

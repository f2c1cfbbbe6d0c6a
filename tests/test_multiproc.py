"""Multi-process paths on CPU (gloo, world_size 2, 127.0.0.1): the bench's max-over-ranks step
time and the torchrun launch of the reference arm (rank 0 runs and prints one JSON line, the
other ranks exit 0 without work).  bench.py --gpus N on GPUs runs one independent replica per
rank, so the job-level logic is exactly this."""
import json
import os
import socket
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    import torch.distributed as dist
    sys.path.insert(0, ROOT)
    import bench
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    v = bench.max_over_ranks(1.5 + rank, world, "cpu")
    out[rank] = v
    dist.destroy_process_group()


def test_max_over_ranks_gloo_two_ranks():
    import torch.multiprocessing as mp
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    assert out[0] == out[1] == 2.5


def test_reference_arm_under_torchrun_two_ranks():
    env = dict(os.environ, CUDA_VISIBLE_DEVICES="")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--impl", "reference",
           "--gpus", "2", "--size", "32", "--steps", "1", "--warmup", "0"]
    p = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=300)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [l for l in p.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle"


def test_sweep_share_partitions_the_problems():
    """cfg5's epsilon sweep over N ranks: every problem solved exactly once, round-robin."""
    sys.path.insert(0, ROOT)
    import bench
    for world in range(1, 9):
        shares = [bench.sweep_share(len(bench.CFG5_EPS), r, world) for r in range(world)]
        flat = sorted(i for sh in shares for i in sh)
        assert flat == list(range(len(bench.CFG5_EPS)))
        assert max(len(sh) for sh in shares) == -(-len(bench.CFG5_EPS) // world)


def test_batch1d_reference_arm_and_rank_slices():
    """cfg1-batch: the reference arm (the oracle over a bounded sample) prints one line; each
    rank's slice of the global problem sequence is disjoint and reproducible."""
    sys.path.insert(0, ROOT)
    import bench
    env = dict(os.environ, CUDA_VISIBLE_DEVICES="")
    p = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--config", "cfg1-batch", "--batch", "32",
                        "--steps", "1", "--warmup", "0"], cwd=ROOT, env=env, capture_output=True, text=True,
                       timeout=300)
    assert p.returncode == 0, p.stderr[-2000:]
    d = json.loads([l for l in p.stdout.splitlines() if l.startswith("{")][-1])
    assert d["impl"] == "reference" and d["value"] > 0 and d["cpu_baseline"]["kind"] == "oracle"
    e_all = bench.batch1d_inputs(64, 0)
    e0, e1 = bench.batch1d_inputs(32, 0), bench.batch1d_inputs(32, 32)
    assert (e_all[:32] == e0).all() and (e_all[32:] == e1).all()
    assert (1e-8 <= e_all).all() and (e_all <= 1e-2).all()


def _plan_worker(rank, world, port, N, out):
    """One rank of the row-strip orchestration on CPU (gloo): it knows only its own [j0, j1) from
    the default partition, gathers the others' like spp_create_dist does, builds its own
    exchange schedule, and the ranks cross-check that every block one sends is the block the
    other receives, in the same position of the same step."""
    import numpy as np
    import torch.distributed as dist
    sys.path.insert(0, ROOT)
    import paper_2108_13468_b200 as spp
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    J = spp.spp_strip_partition(N, world)
    mine = (int(J[rank]), int(J[rank + 1]))
    got = [None] * world
    dist.all_gather_object(got, mine)
    Jg = [g[0] for g in got] + [got[-1][1]]
    plan = spp.spp_dist_plan(N, world, np.array(Jg, np.int32), 2, 64, 56, rank)
    plans = [None] * world
    dist.all_gather_object(plans, plan.tolist())
    ok = list(Jg) == list(J)
    for a in range(world):
        for b in range(world):
            if a == b:
                continue
            sends = [tuple(x) for x in plans[a] if x[1] == a and x[2] == b]
            recvs = [tuple(x) for x in plans[b] if x[1] == a and x[2] == b]
            ok = ok and sends == recvs and len(sends) > 0
    out[rank] = (ok, len(plan))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_row_strip_schedule_matches_across_ranks_gloo(world):
    import torch.multiprocessing as mp
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_plan_worker, args=(world, _free_port(), 512, out), nprocs=world, join=True)
    assert all(out[r][0] for r in range(world)), dict(out)
    assert all(out[r][1] > 0 for r in range(world))

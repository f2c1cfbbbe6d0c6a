"""The one-strip-per-PROCESS path (spp_create_dist) on a one-GPU box.

The real NCCL refuses two ranks on one device, so these tests point SPP_NCCL_LIB at
tests/mock_nccl (a host-staged shared-file transport behind the same ten entry points; test
infrastructure only) and launch the ranks with torchrun, all on cuda:0 with gloo as the process
group.  Everything else is the product path: each process creates its own strip context from
its rows alone, the setup's coefficient all-gather, the exchange lists, the staging of
non-contiguous blocks and the grouped send / receive calls in list order.  No kernel of one rank
waits on another's (all waiting is on the host), so sharing the device is safe.  A functional
check, never a measurement.

Bar (as tests/test_gpu_dist.py): the gathered solution equals the single-GPU solve to 1e-12
relative l2 with identical iteration and corner-cycle counts."""
import json
import os
import shutil
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
MOCK_DIR = os.path.join(ROOT, "tests", "mock_nccl")
MOCK_SRC = os.path.join(MOCK_DIR, "mock_nccl.cpp")
MOCK_SO = os.path.join(MOCK_DIR, "libmock_nccl.so")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.fixture(scope="module")
def mock_env():
    if not os.path.exists(MOCK_SO) or os.path.getmtime(MOCK_SO) < os.path.getmtime(MOCK_SRC):
        gxx = shutil.which("g++")
        if gxx is None:
            pytest.skip("g++ not available to build the mock transport")
        cuda = os.environ.get("CUDA_HOME", "/usr/local/cuda")
        subprocess.run([gxx, "-O2", "-shared", "-fPIC", "-std=c++17", f"-I{cuda}/include", MOCK_SRC, "-o", MOCK_SO,
                        f"-L{cuda}/lib64", "-lcudart", "-lpthread"], check=True)
    return dict(os.environ, SPP_NCCL_LIB=MOCK_SO, SPP_BENCH_SHARED_GPU="1")


def _torchrun(world, script_args, env, timeout=600):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(world),
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port())] + script_args
    return subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=timeout)


@pytest.mark.parametrize("world,cfg,N", [(2, "cfg4", 256), (3, "cfg3", 256), (4, "cfg4", 512), (2, "cfg2", 128)])
def test_strips_one_process_per_rank(mock_env, world, cfg, N):
    p = _torchrun(world, ["tools/nccl_strips_check.py", str(N), cfg], mock_env)
    assert p.returncode == 0, (p.stdout[-2000:], p.stderr[-3000:])
    assert "-> OK" in p.stdout, p.stdout[-2000:]


def test_bench_row_strips_under_torchrun(mock_env):
    """bench.py --gpus 2 as the driver launches it: one JSON line from rank 0, the row-strip
    decomposition of one solve, every timed solve converged (bench.py asserts it)."""
    p = _torchrun(2, ["bench.py", "--gpus", "2", "--size", "512", "--steps", "2", "--warmup", "1",
                      "--no-cpu-baseline"], mock_env)
    assert p.returncode == 0, (p.stdout[-2000:], p.stderr[-3000:])
    lines = [l for l in p.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "strong" and d["value"] > 0
    assert "row strips over 2 GPUs" in d["config"]["parallelism"]
    assert d["exchange"]["blocks_per_solve"] > 0
    assert d["e2e"]["value"] > 0 and d["gpu_launches"] > 0
    assert d["config"]["true_res_jacobi_rel"] <= 1e-8


def test_real_nccl_resolves_and_creates_a_communicator():
    """The real libnccl (torch's, found by the binding) through the library's run-time loader:
    every entry point dist.cu needs resolves, and a one-rank communicator is created and
    destroyed.  (In a subprocess: the loader caches one NCCL per process, and the tests above
    run with the mock.)"""
    code = ("import torch, paper_2108_13468_b200 as spp\n"
            "torch.cuda.set_device(0)\n"
            "spp._nccl_env()\n"
            "import os; print('lib', os.environ.get('SPP_NCCL_LIB'))\n"
            "uid = spp.nccl_unique_id()\n"
            "comm = spp.nccl_comm_create(uid, 1, 0)\n"
            "assert comm\n"
            "spp.nccl_comm_destroy(comm)\n"
            "print('REAL NCCL OK')\n")
    env = {k: v for k, v in os.environ.items() if k not in ("SPP_NCCL_LIB", "SPP_BENCH_SHARED_GPU")}
    p = subprocess.run([sys.executable, "-c", code], cwd=ROOT, env=env, capture_output=True, text=True, timeout=300)
    assert p.returncode == 0 and "REAL NCCL OK" in p.stdout, (p.stdout[-1000:], p.stderr[-2000:])
    assert "mock" not in p.stdout


def test_lost_peer_is_an_error_not_a_hang(mock_env):
    """Failure detection: a rank that leaves before the solve makes the other's solve
    return SPP_E_NCCL (the transport's timeout here; over the real NCCL the library's own
    stream-wait timeout SPP_NCCL_TIMEOUT_S and ncclCommGetAsyncError polling) instead of hanging."""
    env = dict(mock_env, SPP_MOCK_NCCL_TIMEOUT_S="5", SPP_NCCL_TIMEOUT_S="20")
    p = _torchrun(2, ["tests/dist_fail_worker.py"], env, timeout=240)
    assert "LOST PEER DETECTED" in p.stdout, (p.stdout[-2000:], p.stderr[-3000:])
    assert "UNEXPECTED" not in p.stdout

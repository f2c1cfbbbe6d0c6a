#!/usr/bin/env python
"""Benchmark of the hot path: one step = one full preconditioned FGMRES solve of a BASELINE
workload (setup of the coefficients / line factors / multigrid levels + the solve), the
paper's time-to-solution.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config cfg4]

Default workload: cfg4 (B:10), 4096^2 Shishkin mesh, eps = 1e-8, variable convection, seeded
random f, Jacobi-weighted rtol 1e-8.  Prints ONE JSON line (rank 0).
For N > 1 (torchrun) the one cfg4 solve is split into row strips, one per GPU, over NCCL
(strong scaling).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

import spp_inputs as si  # noqa: E402

BASELINE = json.loads((ROOT / "BASELINE.json").read_text())
METRIC = BASELINE["metric"]
UNIT = "unknowns/s"
# Test hook (tests/test_gpu_dist_proc.py): every rank of a torchrun job on cuda:0 with gloo as the
# process group, so the row-strip branch of this file runs on a one-GPU box (with SPP_NCCL_LIB
# pointing at the tests' mock transport).  A functional check, never a measurement.
SHARED_GPU = os.environ.get("SPP_BENCH_SHARED_GPU", "") == "1"


def _peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def _args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg4", help="cfg1..cfg5, or cfg5-sweep (the five eps values as "
                    "independent problems over the ranks)")
    ap.add_argument("--max-iters", type=int, default=None,
                    help="FGMRES cap (cfg5-sweep: common cap, default 100, SURVEY A19; else the library default)")
    ap.add_argument("--restart", type=int, default=0,
                    help="FGMRES(m) restart length (0 = none, the paper; DESIGN.md reading R23)")
    ap.add_argument("--batch", type=int, default=16384, help="cfg1-batch: problems per GPU")
    ap.add_argument("--n", "--size", dest="n", type=int, default=None, help="override N (diagnostics only)")
    ap.add_argument("--eps", type=float, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--profile-all", action="store_true", help="print the per-class profile to stderr")
    return ap.parse_args()


def _workload(cfg):
    return (f"{cfg.name}: -eps Lap u - c.grad u + r u = f, {cfg.N}x{cfg.N} Shishkin mesh "
            f"(sigma=2, beta=1), eps={cfg.eps:g}, Jacobi-weighted rtol {cfg.tol:g}, fp64")


# ---------------------------------------------------------------------------- clocks
class Clocks:
    """nvidia-smi sampled every 200 ms DURING the timed region (B200_PROFILING.md)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.idx = gpu_index
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.p = None

    def start(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                       "-lms", "200", "-i", str(self.idx)], stdout=self.f,
                                      stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return None
        time.sleep(0.25)
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except Exception:
            self.p.kill()
        self.f.flush()
        rows = []
        for line in Path(self.f.name).read_text().splitlines():
            parts = [s.strip() for s in line.split(",")]
            if len(parts) >= 9:
                rows.append(parts)
        os.unlink(self.f.name)
        if not rows:
            return None
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows for k in range(4) if r[5 + k].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


# ---------------------------------------------------------------------------- reference arm
def run_reference(args, rank, world):
    """The oracle, as it stands, on the host cores (the CPU reference arm of this tier)."""
    if rank != 0:
        return None
    import oracle
    if args.config == "cfg1-batch":
        eps = batch1d_inputs(args.batch, 0)
        for _ in range(args.warmup):
            batch1d_oracle_sample(eps, 0, seconds=1.0)
        t0, done = time.perf_counter(), 0
        for _ in range(args.steps):
            d, _, _ = batch1d_oracle_sample(eps, 0, seconds=10.0)
            done += d
        dt = time.perf_counter() - t0
        val = done * (BATCH_N - 1) / dt
        return {"metric": METRIC, "value": val, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": dt * 1e3 / args.steps, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
                "config": {"workload": f"cfg1-batch (bounded sample of the {args.batch}-problem batch)"},
                "cpu_baseline": {"value": val, "unit": UNIT, "cores": 1, "host_cores": os.cpu_count(), "kind": "oracle",
                                 "sample": f"{done} problems of the batch in {args.steps} steps of ~10 s"},
                "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    cfg = si.config(args.config, N=args.n, eps=args.eps)
    N = cfg.N
    x = oracle.mesh(N, cfg.eps, cfg.sigma, cfg.beta_x)
    y = oracle.mesh(N, cfg.eps, cfg.sigma, cfg.beta_y)
    c1, c2, r, f = si.sample_2d(cfg, x, y)

    def step():
        P = oracle.Oracle2D(N, cfg.eps, x, y, c1, c2, r)      # setup
        res = P.solve(f, weighted=cfg.weighted, stop_abs=cfg.stop_abs, tol=cfg.tol)
        P.close()
        return res

    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        res = step()
    dt = (time.perf_counter() - t0) / args.steps
    val = cfg.unknowns / dt
    line = {"metric": METRIC, "value": val, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
            "config": {"workload": _workload(cfg), "N": N, "unknowns": cfg.unknowns, "iters": res["iters"]},
            "cpu_baseline": {"value": val, "unit": UNIT, "cores": 1, "host_cores": os.cpu_count(), "kind": "oracle",
                             "sample": f"one full {cfg.name} solve (setup + FGMRES, {res['iters']} iterations) "
                                       f"per step, single-threaded C oracle"},
            "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    return line


# ---------------------------------------------------------------------------- batched 1D
BATCH_N, BATCH_EPS, BATCH_SEED, BATCH_MAXIT = 256, (1e-8, 1e-2), 7, 64


def batch1d_inputs(nprob, first=0):
    """cfg1-batch: nprob cfg1-sized 1D problems (N = 256), eps log-uniform
    in [1e-8, 1e-2], seeded coefficients / rhs (spp_inputs.sample_batch1d); problems
    first .. first+nprob-1 of the global sequence (each rank its own slice)."""
    _, eps_all = si.batch1d_params(first + nprob, BATCH_SEED, (BATCH_N,), BATCH_EPS)
    eps = eps_all[first:]
    return eps


def _batch_arrays(eps, first, mesh):
    xs, cs, rs, fs = [], [], [], []
    for k, e in enumerate(eps):
        x = mesh(BATCH_N, float(e), 2.0, 1.0)
        c, r, f = si.sample_batch1d(first + k, x, BATCH_SEED)
        xs.append(x); cs.append(c); rs.append(r); fs.append(f)
    return [np.concatenate(a) for a in (xs, cs, rs, fs)]


def batch1d_oracle_sample(eps, first, seconds=15.0):
    """The oracle's 1D GMRES over a bounded sample of the batch (as many problems as fit in
    ~`seconds` of single-threaded CPU time)."""
    import oracle
    t0, done, its = time.perf_counter(), 0, []
    for k, e in enumerate(eps):
        x = oracle.mesh(BATCH_N, float(e), 2.0, 1.0)
        c, r, f = si.sample_batch1d(first + k, x, BATCH_SEED)
        res = oracle.solve1d(BATCH_N, float(e), x, c, r, f, tol=1e-10, maxit=BATCH_MAXIT)
        its.append(res["iters"])
        done += 1
        if time.perf_counter() - t0 > seconds:
            break
    dt = time.perf_counter() - t0
    return done, dt, its


def run_batch1d(args, rank, world):
    import torch
    import paper_2108_13468_b200 as spp

    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", "0")))
    torch.cuda.set_device(dev)
    P, first = args.batch, rank * args.batch
    eps = batch1d_inputs(P, first)
    xcat, ccat, rcat, fcat = _batch_arrays(eps, first, spp.spp_shishkin_mesh)
    Ns = np.full(P, BATCH_N, np.int32)
    d_c, d_r, d_f = [torch.from_numpy(a).to(dev) for a in (ccat, rcat, fcat)]
    u = torch.empty_like(d_f)
    o = spp.spp_default_options(1)
    o.max_iters = BATCH_MAXIT
    stream = torch.cuda.current_stream(dev)
    unknowns = P * (BATCH_N - 1)

    B = spp.Batch1D(Ns, eps, xcat, d_c, d_r, options=o, stream=stream)   # workspace + first setup

    def step(c_, r_, f_, u_):
        n0 = B.launches()
        B.setup(c_, r_)                  # setup counted in time-to-solution
        res = B.solve(f_, u_)
        return res, B.launches() - n0

    for _ in range(args.warmup):
        res, _ = step(d_c, d_r, d_f, u)
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    clk = Clocks(dev.index)
    clk.start()
    launches = 0
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        res, n = step(d_c, d_r, d_f, u)
        launches += n
    e1.record(stream)
    torch.cuda.synchronize()
    clocks = clk.stop()
    ms = max_over_ranks(e0.elapsed_time(e1) / args.steps, world, dev)
    solve_ms = res.stats["solve_s"] * 1e3
    e2e = None
    if not args.no_e2e:
        hp = [torch.from_numpy(a).pin_memory() for a in (ccat, rcat, fcat)]
        hu = torch.empty(unknowns, dtype=torch.float64).pin_memory()
        step(hp[0], hp[1], hp[2], hu)
        if world > 1:
            torch.distributed.barrier()
        t0 = time.perf_counter()
        for _ in range(max(1, min(args.steps, 3))):
            step(hp[0], hp[1], hp[2], hu)
        ems = max_over_ranks((time.perf_counter() - t0) * 1e3 / max(1, min(args.steps, 3)), world, dev)
        e2e = {"value": unknowns * world / (ems * 1e-3), "unit": UNIT, "h2d_bytes_per_step": 3 * unknowns * 8,
               "d2h_bytes_per_step": unknowns * 8, "ms_per_step": ems}
    if rank != 0:
        return None
    peak, peak_kind = _peaks()
    # dominant kernel k_solve1d_batch: algorithmic bytes = inputs c, r, f read + u written
    # (32 B/node); the Krylov basis stays in L1/L2 per CTA
    alg = 32.0 * unknowns
    line = {
        "metric": METRIC, "value": unknowns * world / (ms * 1e-3), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"cfg1-batch: {P} independent 1D problems per GPU (N={BATCH_N}, eps log-uniform "
                               f"{BATCH_EPS}, seeded c, r, f), right FGMRES, Jacobi-weighted rtol 1e-10, fp64",
                   "problems_per_s": P * world / (ms * 1e-3), "unknowns": unknowns,
                   "iters": {"min": int(res.iters.min()), "median": float(np.median(res.iters)),
                             "max": int(res.iters.max())}, "converged": int(res.converged.sum()),
                   "setup_s": res.stats["setup_s"], "solve_s": res.stats["solve_s"],
                   "l2": "per-step setup + solve; per-CTA Krylov basis re-read from L1/L2",
                   "parallelism": "replicas: an independent batch per GPU (weak scaling)" if world > 1 else "single GPU"},
        "roofline": {"kernel": "k_solve1d_batch", "bound": "hbm", "achieved": alg / (solve_ms * 1e-3) / 1e9,
                     "peak": peak, "unit": "GB/s", "frac": alg / (solve_ms * 1e-3) / 1e9 / peak, "traffic": None,
                     "peak_kind": peak_kind, "avg_launch_ms": solve_ms, "algorithmic_bytes_per_launch": alg},
        "gpu_launches": int(launches // max(args.steps, 1)),
        "clocks": clocks,
    }
    if e2e:
        line["e2e"] = e2e
    if not args.no_cpu_baseline:
        done, dt, its = batch1d_oracle_sample(eps, first)
        line["cpu_baseline"] = {"value": done * (BATCH_N - 1) / dt, "unit": UNIT, "cores": 1, "host_cores": os.cpu_count(), "kind": "oracle",
                                "sample": f"the first {done} problems of the batch, {dt:.1f} s"}
    return line


# ---------------------------------------------------------------------------- our arm
def max_over_ranks(ms, world, device):
    """The step time of the job: the maximum over ranks (one value per rank, all_reduce MAX on the
    process group; gloo on CPU tensors in the tests, NCCL on the GPU in the bench)."""
    if world <= 1:
        return ms
    import torch
    if torch.distributed.get_backend() == "gloo":
        device = "cpu"
    t = torch.tensor([float(ms)], dtype=torch.float64, device=device)
    torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    return float(t.item())


def cpu_baseline(cfg):
    """The oracle timed on this host on a bounded sample: one full solve of the same workload
    (~10 s of single-threaded CPU work at 4096^2)."""
    import oracle
    N = cfg.N
    x = oracle.mesh(N, cfg.eps, cfg.sigma, cfg.beta_x)
    y = oracle.mesh(N, cfg.eps, cfg.sigma, cfg.beta_y)
    c1, c2, r, f = si.sample_2d(cfg, x, y)
    t0 = time.perf_counter()
    P = oracle.Oracle2D(N, cfg.eps, x, y, c1, c2, r)
    res = P.solve(f, weighted=cfg.weighted, stop_abs=cfg.stop_abs, tol=cfg.tol)
    dt = time.perf_counter() - t0
    P.close()
    return {"value": cfg.unknowns / dt, "unit": UNIT, "cores": 1, "host_cores": os.cpu_count(), "kind": "oracle",
            "sample": f"one full {cfg.name} solve (setup + FGMRES, {res['iters']} iterations), {dt:.2f} s"}


CFG5_EPS = [1e-2, 1e-4, 1e-6, 1e-8, 1e-10]   # B:11


def sweep_share(n_items, rank, world):
    """Independent problems of a sweep, round-robin over ranks (no data-path collective)."""
    return [i for i in range(n_items) if i % world == rank]


def run_sweep(args, rank, world):
    """cfg5's epsilon sweep (B:11) as one step: the five independent 8192^2 solves, sharded over
    the ranks round-robin; the step time is the max over ranks.  Common iteration cap for the
    non-converging large-eps cells."""
    import torch
    import paper_2108_13468_b200 as spp

    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", "0")))
    torch.cuda.set_device(dev)
    mine = sweep_share(len(CFG5_EPS), rank, world)
    jobs = []
    for i in mine:
        cfg = si.config("cfg5", N=args.n, eps=CFG5_EPS[i])
        N = cfg.N
        x = spp.spp_shishkin_mesh(N, cfg.eps, cfg.sigma, cfg.beta_x)
        y = spp.spp_shishkin_mesh(N, cfg.eps, cfg.sigma, cfg.beta_y)
        c1, c2, r, f = si.sample_2d(cfg, x, y)
        d = [torch.from_numpy(np.ascontiguousarray(a).ravel()).to(dev) for a in (c1, c2, r, f)]
        o = spp.spp_default_options(2)
        o.tol = cfg.tol
        o.max_iters = args.max_iters if args.max_iters is not None else 100
        jobs.append((cfg, x, y, d, torch.empty_like(d[3]), o))

    def step():
        # one problem at a time: create (eps fixes the mesh), set up, solve, free -- a capped
        # non-converging cell keeps 2 x max_iters Krylov vectors of 537 MB alive
        its = {}
        for cfg, x, y, d, u, o in jobs:
            S = spp.Solver(2, cfg.N, cfg.eps, x, y, d[0], d[1], d[2], options=o)
            res = S.solve(d[3], u)
            its[f"{cfg.eps:g}"] = res.stats["iters"]
            S.close()
        return its

    for _ in range(args.warmup):
        step()
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    clk = Clocks(dev.index)
    clk.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        its = step()
    e1.record()
    torch.cuda.synchronize()
    clocks = clk.stop()
    ms = max_over_ranks(e0.elapsed_time(e1) / args.steps, world, dev)
    iters = {}
    if world > 1:
        allits = [None] * world
        torch.distributed.all_gather_object(allits, its)
        for d_ in allits:
            iters.update(d_)
    else:
        iters = its
    if rank != 0:
        return None
    N = si.config("cfg5", N=args.n).N
    total = len(CFG5_EPS) * (N - 1) ** 2
    return {"metric": METRIC, "value": total / (ms * 1e-3), "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"cfg5 epsilon sweep: {len(CFG5_EPS)} independent {N}x{N} solves "
                                   f"(eps {CFG5_EPS}), round-robin over ranks", "N": N,
                       "unknowns": total, "max_iters": args.max_iters,
                       "iters_per_eps": {k: iters[k] for k in sorted(iters, key=float, reverse=True)},
                       "parallelism": f"task-parallel: independent eps problems over {world} GPU(s) (not the "
                                      f"row-strip decomposition of one solve; that is the default --config cfg4)",
                       "l2": "inputs larger than L2"},
            "clocks": clocks}


def nccl_comm(rank, world):
    """An NCCL communicator for the row strips: rank 0 makes the id, torch.distributed carries it."""
    import torch.distributed as dist
    import paper_2108_13468_b200 as spp
    obj = [spp.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    return spp.nccl_comm_create(obj[0], world, rank)


def strip_rows(N, rank, world):
    """This rank's interior rows [j0, j1) of the default row strips (spp_strip_partition)."""
    import paper_2108_13468_b200 as spp
    J = spp.spp_strip_partition(N, world)
    return int(J[rank]), int(J[rank + 1])


def run_ours(args, rank, world):
    """One GPU: spp_create + spp_solve.  N GPUs (torchrun): the row-strip decomposition of the
    same solve, one strip per rank over NCCL (strong scaling: the
    job solves the one cfg4 problem)."""
    import torch
    import paper_2108_13468_b200 as spp

    dev = torch.device("cuda", 0 if SHARED_GPU else int(os.environ.get("LOCAL_RANK", "0")))
    torch.cuda.set_device(dev)
    cfg = si.config(args.config, N=args.n, eps=args.eps)
    N, m = cfg.N, cfg.N - 1
    x = spp.spp_shishkin_mesh(N, cfg.eps, cfg.sigma, cfg.beta_x)
    y = spp.spp_shishkin_mesh(N, cfg.eps, cfg.sigma, cfg.beta_y)
    c1, c2, r, f = si.sample_2d(cfg, x, y)
    j0, j1 = strip_rows(N, rank, world) if world > 1 else (1, N)
    rows = slice(j0 - 1, j1 - 1)                         # this rank's rows of the (N-1)^2 grid
    host = [np.ascontiguousarray(a[rows]).ravel() for a in (c1, c2, r, f)]
    nloc = (j1 - j0) * m
    d_c1, d_c2, d_r, d_f = [torch.from_numpy(a).to(dev) for a in host]
    u = torch.empty_like(d_f)
    o = spp.spp_default_options(2)
    o.stop = spp.SPP_STOP_REL_JACOBI if cfg.weighted else (spp.SPP_STOP_ABS_L2 if cfg.stop_abs else spp.SPP_STOP_REL_L2)
    o.tol = cfg.tol
    if args.max_iters is not None:
        o.max_iters = args.max_iters
    o.restart = args.restart
    stream = torch.cuda.current_stream(dev)
    comm = None
    if world > 1:
        comm = nccl_comm(rank, world)
        S = spp.DistSolver(N, cfg.eps, x, y, d_c1, d_c2, d_r, j0, j1, comm, rank, world, options=o, stream=stream)
    else:
        S = spp.Solver(2, N, cfg.eps, x, y, d_c1, d_c2, d_r, options=o, stream=stream)

    nsolves = [0]

    def step(c1_, c2_, r_, f_, u_):
        nsolves[0] += 1
        S.setup(c1_, c2_, r_)
        return S.solve(f_, u_)

    def check(res):
        """every timed solve must converge (ADVICE: a non-converged solve is not a valid step)"""
        assert res.status == spp.SPP_OK and res.stats["converged"] == 1, res.stats

    # warm-up exactly as the timed steps run (this also captures the corner-solve CUDA graph),
    # then one more untimed step with every kernel class profiled, to find the dominant class
    res = None
    for _ in range(max(1, args.warmup)):      # at least one (its iteration count is the reference)
        res = step(d_c1, d_c2, d_r, d_f, u)
        check(res)
    iters_ref = res.stats["iters"]
    S.profile_reset()
    S.profile_enable(1)
    res = step(d_c1, d_c2, d_r, d_f, u)
    prof_all = S.profile()
    prof = {k: v for k, v in prof_all.items() if k not in ("exchange",)}
    dom = max(prof, key=lambda k: prof[k]["ms"])
    dom_idx = list(prof_all).index(dom)
    tot_ms = sum(v["ms"] for v in prof_all.values())
    if args.profile_all and rank == 0:
        for k, v in prof_all.items():
            if v["launches"]:
                print(f"[prof] {k:18s} launches={v['launches']:6d} ms={v['ms']:9.3f} ({100*v['ms']/tot_ms:5.1f}%) "
                      f"GB/s={v['bytes']/max(v['ms'],1e-9)/1e6:8.1f}", file=sys.stderr)
    # per-class roofline fractions (north_star: stencil, smoother and vector kernels), from the
    # profiled step's CUDA events: algorithmic bytes / device time
    peak, peak_kind = _peaks()
    classes = {}
    for k, v in prof_all.items():
        if v["launches"] and v["ms"] > 0:
            gbs = v["bytes"] / (v["ms"] * 1e-3) / 1e9
            classes[k] = {"launches": v["launches"], "ms": round(v["ms"], 4), "share": round(v["ms"] / tot_ms, 4),
                          "achieved_gbs": round(gbs, 1), "frac": round(gbs / peak, 4)}
    S.profile_reset()
    S.profile_enable(0)          # the timed region runs exactly as a user's solve (no event brackets)

    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    clk = Clocks(dev.index)
    clk.start()
    l0 = S.kernel_launches()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    results = []
    e0.record(stream)
    for _ in range(args.steps):
        results.append(step(d_c1, d_c2, d_r, d_f, u))
    e1.record(stream)
    torch.cuda.synchronize()
    clocks = clk.stop()
    for rr in results:
        check(rr)
        assert rr.stats["iters"] == iters_ref, (rr.stats["iters"], iters_ref)
    res = results[-1]
    launches = S.kernel_launches() - l0
    ms = max_over_ranks(e0.elapsed_time(e1) / args.steps, world, dev)
    if world > 1:
        torch.distributed.barrier()
    # roofline pass: the same steps again with CUDA events bracketing every launch of the dominant
    # kernel class (on the library's stream), for its average launch duration
    S.profile_reset()
    S.profile_enable(1 << dom_idx)
    for _ in range(args.steps):
        step(d_c1, d_c2, d_r, d_f, u)
    torch.cuda.synchronize()
    prof = S.profile()[dom]
    S.profile_enable(0)

    # e2e: the same step through the public API with pinned HOST buffers (H2D of c1, c2, r, f
    # and D2H of u inside the timed region)
    e2e = None
    if not args.no_e2e:
        hp = [torch.from_numpy(a).pin_memory() for a in host]
        hu = torch.empty(nloc, dtype=torch.float64).pin_memory()
        step(hp[0], hp[1], hp[2], hp[3], hu)
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        t0 = time.perf_counter()
        e0.record(stream)
        ne = max(1, min(args.steps, 3))
        for _ in range(ne):
            step(hp[0], hp[1], hp[2], hp[3], hu)
        e1.record(stream)
        torch.cuda.synchronize()
        ems = max_over_ranks(max(e0.elapsed_time(e1), (time.perf_counter() - t0) * 1e3) / ne, world, dev)
        e2e = {"value": cfg.unknowns / (ems * 1e-3), "unit": UNIT,
               "h2d_bytes_per_step": 4 * nloc * 8, "d2h_bytes_per_step": nloc * 8, "ms_per_step": ems}
    info = S.dist_info()
    S.close()
    if comm is not None:
        spp.nccl_comm_destroy(comm)

    if rank != 0:
        return None
    avg_ms = prof["ms"] / max(prof["launches"], 1)
    avg_bytes = prof["bytes"] / max(prof["launches"], 1)
    achieved = avg_bytes / (avg_ms * 1e-3) / 1e9 if avg_ms > 0 else 0.0
    traffic = None
    tf = ROOT / "profiles" / "traffic.json"
    if tf.exists() and world == 1:
        try:
            traffic = json.loads(tf.read_text()).get(f"{cfg.name}:{dom}")
        except Exception:
            traffic = None
    line = {
        "metric": METRIC, "value": cfg.unknowns / (ms * 1e-3), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": _workload(cfg), "N": N, "unknowns": cfg.unknowns,
                   "iters_per_solve": res.stats["iters"],
                   **({"restart": args.restart} if args.restart else {}),
                   "mg_cycles_per_apply": [res.stats["mg_cycles_min"], res.stats["mg_cycles_max"]],
                   "time_to_solution_s": ms * 1e-3, "setup_s": res.stats["setup_s"],
                   "true_res_jacobi_rel": res.stats["true_res_jacobi_rel"],
                   "l2": "inputs larger than L2 (each grid function 134 MB > 126 MB L2)",
                   "parallelism": (f"row strips over {world} GPUs (NCCL; rows [{j0},{j1}) on rank 0; "
                                   f"{info['strip_levels']} corner levels on strips)"
                                   + ("; SHARED-GPU FUNCTIONAL CHECK, NOT A MEASUREMENT" if SHARED_GPU else ""))
                                  if world > 1 else "single GPU"},
        "roofline": {"kernel": dom, "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "traffic_source": "profiles/traffic.json (ncu --set full capture of this kernel class)"
                                       if traffic is not None else None,
                     "peak_kind": peak_kind, "avg_launch_ms": avg_ms, "algorithmic_bytes_per_launch": avg_bytes,
                     "classes": classes},
        "gpu_launches": int(launches // max(args.steps, 1)),
        "clocks": clocks,
    }
    if world > 1:
        line["exchange"] = {"blocks_per_solve": info["xfers"] / nsolves[0], "MB_per_solve": info["bytes"] / nsolves[0] / 1e6,
                            "steps_per_solve": info["exchanges"] / nsolves[0],
                            "note": "rank 0's NCCL send/recv blocks incl. the setup's coefficient all-gather; the "
                                    "'exchange' class in roofline.classes is its device time"}
    if e2e:
        line["e2e"] = e2e
    if not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(cfg)
    return line


def main():
    args = _args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist
        backend = "nccl" if torch.cuda.is_available() and not SHARED_GPU else "gloo"
        if backend == "nccl":
            torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
        dist.init_process_group(backend)
    if args.config == "cfg5-sweep" and args.impl != "reference":
        line = run_sweep(args, rank, world)
    elif args.config == "cfg1-batch" and args.impl != "reference":
        line = run_batch1d(args, rank, world)
    else:
        line = run_reference(args, rank, world) if args.impl == "reference" else run_ours(args, rank, world)
    if rank == 0 and line is not None:
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

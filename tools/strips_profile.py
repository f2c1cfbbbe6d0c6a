"""What the row-strip decomposition costs, measured on ONE GPU with the loopback
transport (spp_create_strips): P = 1, 2, 4, 8 strips of the cfg4 solve run one after another on
the same device, so the device time is the SUM over the strips of every phase.

Per P: the serialised device time per solve (setup + solve; CUDA events), iteration and
corner-cycle counts, the per-class profile (the 'exchange' class = the loopback copies), the
number of exchange steps / blocks / bytes per solve, and the redundant work the decomposition
adds = serialised time(P) - time(1).  NOT a multi-GPU measurement: it bounds the work each of P
GPUs would do (serialised / P if the phases divided evenly) and counts the messages NCCL would
carry; the sequential phases (M_II across the top strips) do not divide.

    python tools/strips_profile.py [N] [P,P,...] > gpurun_out/strips_profile.txt

With strips the per-class profile is the FIRST strip's (a bottom strip: no M_II), i.e. the work one
rank keeps, plus every loopback copy of the job in the 'exchange' class.
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2108_13468_b200 as spp  # noqa: E402
import spp_inputs as si  # noqa: E402


def main():
    N = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
    torch.cuda.set_device(0)
    cfg = si.config("cfg4", N=N)
    x = spp.spp_shishkin_mesh(N, cfg.eps, cfg.sigma, cfg.beta_x)
    y = spp.spp_shishkin_mesh(N, cfg.eps, cfg.sigma, cfg.beta_y)
    c1, c2, r, f = si.sample_2d(cfg, x, y)
    d = [torch.from_numpy(np.ascontiguousarray(a).ravel()).cuda() for a in (c1, c2, r, f)]
    u = torch.empty_like(d[3])
    o = spp.spp_default_options(2)
    o.stop = spp.SPP_STOP_REL_JACOBI
    o.tol = cfg.tol
    base = None
    uref = None
    print(f"# cfg4 N={N} eps={cfg.eps:g}: P strips on one device, loopback transport (serialised)")
    Ps = [int(t) for t in sys.argv[2].split(",")] if len(sys.argv) > 2 else [1, 2, 4, 8]
    for P in Ps:
        S = spp.Solver(2, N, cfg.eps, x, y, d[0], d[1], d[2], options=o, strips=P)

        def step():
            S.setup(d[0], d[1], d[2])
            return S.solve(d[3], u)

        for _ in range(3):
            res = step()
        S.profile_reset()
        S.profile_enable(1)
        step()
        prof = S.profile()
        S.profile_reset()
        S.profile_enable(0)
        info0 = S.dist_info() if P > 1 else None
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        K = 5
        e0.record()
        for _ in range(K):
            res = step()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / K
        if P == 1:
            base, uref = ms, u.clone()
            rel = 0.0
        else:
            rel = float(torch.linalg.norm(u - uref) / torch.linalg.norm(uref))
        line = (f"P={P}: {ms:8.3f} ms per solve serialised ({ms / base:5.2f}x one GPU; {ms / P:7.3f} ms = 1/P of it), "
                f"iters {res.stats['iters']}, cycles {res.stats['mg_cycles_total']}, rel. diff to P=1 {rel:.2e}")
        if P > 1:
            info1 = S.dist_info()
            n = K
            line += (f"; per solve: {(info1['exchanges'] - info0['exchanges']) / n:.0f} exchange steps, "
                     f"{(info1['xfers'] - info0['xfers']) / n:.0f} blocks, "
                     f"{(info1['bytes'] - info0['bytes']) / n / 1e6:.1f} MB, strip levels {info1['strip_levels']}")
        print(line)
        tot = sum(v["ms"] for v in prof.values())
        for k, v in prof.items():
            if v["launches"]:
                print(f"      {k:18s} launches={v['launches']:6d} ms={v['ms']:8.3f} ({100 * v['ms'] / tot:5.1f}%)")
        S.close()
        del S


if __name__ == "__main__":
    main()

"""Race check of the lock-free hand-offs (SURVEY §5 race detection).

    python tools/stress_check.py save  OUT.npz      # with the normal library
    python tools/stress_check.py check OUT.npz [R]  # with the SPP_STRESS library, R repetitions

The cases run every hand-off of the downstream sweep (k_wave): the edge rings between the warps
of a tile, the write-back / TMA staging slots, the chained M_II strips through global memory and
the row-strip relays, in whole solves and through the stage hooks.  The stress build sleeps a
pseudo-random time at every hand-off point, so producer / consumer orders differ from run to
run; every output must be bit-for-bit the normal build's.  Exit status 1 on any difference."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2108_13468_b200 as spp  # noqa: E402
import spp_inputs as si  # noqa: E402


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64).ravel()).cuda()


def cases():
    out = {}
    for name, N, eps, strips in [("cfg4", 1024, 1e-8, 1), ("cfg4", 512, 1e-4, 1), ("cfg5", 2048, 1e-6, 1),
                                 ("cfg3", 1024, 1e-6, 1), ("cfg4", 1024, 1e-8, 4), ("cfg4", 4096, 1e-8, 1)]:
        cfg = si.config(name, N=N, eps=eps)
        x = spp.spp_shishkin_mesh(N, cfg.eps, cfg.sigma, cfg.beta_x)
        y = spp.spp_shishkin_mesh(N, cfg.eps, cfg.sigma, cfg.beta_y)
        c1, c2, r, f = si.sample_2d(cfg, x, y)
        o = spp.spp_default_options(2)
        o.tol = cfg.tol
        S = spp.Solver(2, N, cfg.eps, x, y, dev(c1), dev(c2), dev(r), options=o, strips=strips)
        res = S.solve(dev(f))
        key = f"{name}_{N}_{eps:g}_P{strips}"
        out[key + "_u"] = res.u.cpu().numpy()
        out[key + "_hist"] = np.asarray(res.hist)
        out[key + "_counts"] = np.array([res.stats["iters"], res.stats["mg_cycles_total"]])
        print(f"  {key}: solve {1e3 * res.stats['solve_s']:.2f} ms (device time)")
        if strips == 1 and N == 1024:
            m = N - 1
            q = si.random_field(3, (m, m))
            z = torch.zeros(m * m, dtype=torch.float64, device="cuda")
            S.apply_stage("MII_JACOBI", dev(q), z)                     # the chained exact sweep
            out[key + "_mii"] = z.cpu().numpy()
            for l in range(min(3, S.mg_levels())):                     # tiled certified-halo sweeps
                nl = S.mg_level_n(l)
                b = si.random_field(10 + l, (nl, nl))
                e0 = si.random_field(20 + l, (nl, nl))
                t = dev(e0)
                S.apply_stage("GS_SWEEP", dev(b), t, level=l)
                out[key + f"_gs{l}"] = t.cpu().numpy()
        S.close()
    return out


def main():
    mode, path = sys.argv[1], sys.argv[2]
    print("library:", spp.spp_version())
    if mode == "check":
        assert spp.spp_version().endswith("+stress"), "check mode needs the SPP_STRESS library"
    if mode == "save":
        t0 = time.time()
        out = cases()
        print(f"normal library: {time.time() - t0:.2f} s")
        np.savez(path, **out)
        print("saved", path)
        return 0
    ref = np.load(path)
    reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
    bad = 0
    for rep in range(reps):
        t0 = time.time()
        got = cases()
        print(f"rep {rep}: {time.time() - t0:.2f} s")
        for k in ref.files:
            same = np.array_equal(ref[k], got[k])
            if not same:
                bad += 1
                d = np.max(np.abs(ref[k].astype(float) - got[k].astype(float)))
                print(f"rep {rep}: {k} DIFFERS (max |diff| {d:.3e})")
        print(f"rep {rep}: {len(ref.files)} outputs compared, {bad} differences so far")
    print("STRESS OK" if bad == 0 else "STRESS FAILED")
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())

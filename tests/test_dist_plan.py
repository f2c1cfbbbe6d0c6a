"""Host logic of the row-strip decomposition, no GPU: the default
partition, and the exchange schedule the solve runs (spp_dist_plan uses the solve's own
generators): every block is well formed, and the rows a strip receives in each step are
exactly the halo that step needs -- one row on each side for the stencil, the certified halo
rows above plus one row below for a corner level's smoothing, every other strip's rows for
the all-gathers."""
import numpy as np
import pytest

import paper_2108_13468_b200 as spp

ROLE = dict(V=0, Z=1, U=2, W=3, CHAIN=4, LB=5, LE=6, LQ=7, LG=8, LRHO=9, BC=10, ZC=11, ZC2=12, PART=13)
KRB = 592


def test_default_partition():
    for N in (16, 64, 256, 4096, 8192):
        n = N // 2
        for P in range(1, 9):
            try:
                J = spp.spp_strip_partition(N, P)
            except spp.SppError:
                assert P > 1 and ((P + 1) // 2 > n or (P - (P + 1) // 2 - 1) * 32 >= n - 1)
                continue
            assert J[0] == 1 and J[-1] == N and np.all(np.diff(J) > 0)
            if P > 1:
                assert n + 1 in J                                       # the X/I | C/Y split
                Pb = list(J).index(n + 1)
                assert Pb == (P + 1) // 2
                sizes = np.diff(J)
                assert sizes[:Pb].max() - sizes[:Pb].min() <= 1
                assert all(sz % 32 == 0 for sz in sizes[Pb + 1:])             # M_II relay strips: whole warps
    with pytest.raises(spp.SppError):
        spp.spp_strip_partition(8, 9)


def _rows_received(plan, step, dst, role=None):
    rows = set()
    for b in plan:
        if b[0] != step or b[2] != dst or (role is not None and b[3] != role):
            continue
        first = b[5] // b[9]
        rows.update(range(first, first + b[8]))
    return rows


@pytest.mark.parametrize("N,P,D", [(256, 2, 2), (256, 3, 2), (512, 4, 2), (512, 8, 3), (1024, 5, 1), (4096, 8, 2)])
def test_schedule_blocks_and_halos(N, P, D):
    J = spp.spp_strip_partition(N, P)
    halo, warm = 64, 56
    plan = spp.spp_dist_plan(N, P, J, D, halo, warm, -1)
    assert len(plan) > 0
    n = N // 2
    pitch = -(-(N + 1) // 16) * 16
    for b in plan:
        step, src, dst, role, slot, soff, doff, width, rows, bp, _ = b
        assert src != dst and 0 <= src < P and 0 <= dst < P and rows >= 1 and 1 <= width <= bp
        if role in (ROLE["V"], ROLE["Z"], ROLE["U"]):
            assert bp == pitch and soff == doff
            r0 = soff // pitch
            assert 1 <= r0 and r0 + rows - 1 <= N - 1                   # interior rows only
            assert soff % pitch + width <= pitch
    # the stencil halo (second-to-last Z step): exactly the neighbour rows
    zsteps = sorted({b[0] for b in plan if b[3] == ROLE["Z"]})
    spmv = zsteps[-1]
    for r in range(P):
        want = set()
        if r > 0:
            want.add(J[r] - 1)
        if r < P - 1:
            want.add(J[r + 1])
        assert _rows_received(plan, spmv, r) == want
    # all-gathers of partial sums: P-1 segments in, P-1 out, per rank
    psteps = sorted({b[0] for b in plan if b[3] == ROLE["PART"]})
    for s in psteps:
        for r in range(P):
            ins = [b for b in plan if b[0] == s and b[3] == ROLE["PART"] and b[2] == r]
            outs = [b for b in plan if b[0] == s and b[3] == ROLE["PART"] and b[1] == r]
            assert len(ins) == len(outs) == P - 1
            assert sorted(b[5] // KRB % P for b in ins) == sorted(set(range(P)) - {r})
    # level-0 smoothing rhs: the certified halo rows above and the row below each corner strip
    nD = n >> D
    Cb = [1] + [int(round(r * nD / P)) << D for r in range(1, P)] + [n + 1]
    rsteps = [b[0] for b in plan if b[3] == ROLE["LRHO"] and b[4] == 0]
    step0 = max(rsteps)                                                  # (the corner-in step also moves rho)
    for r in range(P):
        lo, hi = Cb[r], Cb[r + 1]
        want = set(range(hi, min(hi + halo, n + 1))) | ({lo - 1} if r > 0 else set())
        assert _rows_received(plan, step0, r, ROLE["LRHO"]) == want
    # the corner right-hand side reaches every corner strip from the bottom strips' rows
    cin = min(rsteps)
    Pb = list(J).index(n + 1)
    for r in range(P):
        own = set(range(J[r], J[r + 1])) if r < Pb else set()
        got = _rows_received(plan, cin, r, ROLE["BC"])
        assert got | (own & set(range(Cb[r], Cb[r + 1]))) == set(range(Cb[r], Cb[r + 1]))


def test_schedule_rejects_bad_geometry():
    J = spp.spp_strip_partition(512, 6)
    bad = J.copy()
    bad[4] += 1                                                          # a relay strip not of whole warps
    with pytest.raises(spp.SppError):
        spp.spp_dist_plan(512, 6, bad, 2, 64, 56, -1)
    J = spp.spp_strip_partition(256, 4)
    bad = J.copy()
    bad[2] += 1                                                          # no boundary at n+1
    with pytest.raises(spp.SppError):
        spp.spp_dist_plan(256, 4, bad, 2, 64, 56, -1)
    with pytest.raises(spp.SppError):
        spp.spp_dist_plan(256, 4, J, 7, 64, 56, -1)                      # more strip levels than fit

"""GPU parity of the batched 1D solver (spp_batch1d_*) against the oracle's
single-problem 1D GMRES (oracle.solve1d, P:375-386 / P:828-833) on the same seeded inputs:
identical iteration counts and <= 1e-9 relative l2 per problem; and bitwise equality with the
single-problem GPU solve (same kernels' body)."""
import numpy as np
import pytest

import oracle
import spp_inputs as si

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2108_13468_b200 as spp  # noqa: E402


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64).ravel()).cuda()


def rel(a, b):
    a, b = np.asarray(a).ravel(), np.asarray(b).ravel()
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


def build_batch(Ns, eps, sigma=2.0, beta=1.0, sampler=None, seed=7):
    xs, cs, rs, fs = [], [], [], []
    for p, (N, e) in enumerate(zip(Ns, eps)):
        x = spp.spp_shishkin_mesh(int(N), float(e), sigma, beta)
        c, r, f = sampler(p, x) if sampler else si.sample_batch1d(p, x, seed)
        xs.append(x); cs.append(c); rs.append(r); fs.append(f)
    return xs, cs, rs, fs


def offsets(Ns):
    return np.concatenate([[0], np.cumsum(np.asarray(Ns) - 1)])


def oracle_solve(N, e, c, r, f, o, sigma=2.0, beta=1.0):
    return oracle.solve1d(int(N), float(e), oracle.mesh(int(N), float(e), sigma, beta), c, r, f, side=o.side,
                          weighted=1 if o.stop == 0 else 0, stop_abs=1 if o.stop == 2 else 0, tol=o.tol,
                          maxit=o.max_iters)


@pytest.mark.parametrize("device", [True, False])
def test_batch_mixed_sizes_matches_oracle(device):
    Ns = [4, 6, 8, 128, 256, 1000, 2048, 8192, 256, 512, 130, 4096, 64]
    _, eps = si.batch1d_params(len(Ns), seed=11)
    xs, cs, rs, fs = build_batch(Ns, eps)
    o = spp.spp_default_options(1)
    conv = dev if device else (lambda a: np.ascontiguousarray(a))
    B = spp.Batch1D(Ns, eps, np.concatenate(xs), conv(np.concatenate(cs)), conv(np.concatenate(rs)), options=o)
    res = B.solve(conv(np.concatenate(fs)))
    u = res.u.cpu().numpy() if device else res.u
    off = offsets(Ns)
    for p, N in enumerate(Ns):
        orc = oracle_solve(N, eps[p], cs[p], rs[p], fs[p], o)
        assert res.iters[p] == orc["iters"], (p, N, eps[p])
        assert bool(res.converged[p]) == orc["converged"]
        assert rel(u[off[p]:off[p + 1]], orc["u"]) <= 1e-9, (p, N)
        assert abs(res.res[p] - orc["res_final"]) <= 1e-9 * orc["res0"]
    assert res.status == (spp.SPP_OK if res.converged.all() else spp.SPP_NOT_CONVERGED)
    assert res.stats["iters"] == max(res.iters)


def test_batch_equals_single_solves_bitwise():
    Ns = [256] * 6 + [1024] * 3
    _, eps = si.batch1d_params(len(Ns), seed=3)
    xs, cs, rs, fs = build_batch(Ns, eps)
    B = spp.Batch1D(Ns, eps, np.concatenate(xs), dev(np.concatenate(cs)), dev(np.concatenate(rs)))
    u = B.solve(dev(np.concatenate(fs))).u.cpu().numpy()
    off = offsets(Ns)
    # re-setup with the same coefficients from host memory reproduces the result
    B.setup(np.concatenate(cs), np.concatenate(rs))
    assert np.array_equal(B.solve(dev(np.concatenate(fs))).u.cpu().numpy(), u)
    for p in (0, 5, 6, 8):
        S = spp.Solver(1, Ns[p], eps[p], xs[p], None, dev(cs[p]), None, dev(rs[p]))
        us = S.solve(dev(fs[p])).u.cpu().numpy()
        assert np.array_equal(us, u[off[p]:off[p + 1]]), p


def test_batch_table2_paper_mode():
    """Table 2 as ONE batch: left GMRES, true inf-norm stop K N^-1 ln N (K = 1).
    The stop tolerance is per problem in the paper; the batch shares options, so the batch is
    split by N (one tolerance per N)."""
    from conftest import load_table
    t2 = load_table("table2_1d_iters.txt")
    for col, N in enumerate([128, 256, 512, 1024, 2048]):
        eps = [e for e, row in t2.items() if row[col] is not None]
        want = [int(t2[e][col]) for e in eps]
        cfg = si.config("ex1d", N=N)
        xs, cs, rs, fs = build_batch([N] * len(eps), eps, 2.0, 0.99,
                                     sampler=lambda p, x: si.sample_1d(cfg, x))
        o = spp.spp_default_options(1)
        o.side, o.stop, o.tol = spp.SPP_LEFT, spp.SPP_STOP_ABS_MAX, np.log(N) / N
        B = spp.Batch1D([N] * len(eps), eps, np.concatenate(xs), dev(np.concatenate(cs)), dev(np.concatenate(rs)),
                        options=o)
        res = B.solve(dev(np.concatenate(fs)))
        assert list(res.iters) == want, (N, list(res.iters), want)


def test_batch_rejects_bad_inputs():
    x = spp.spp_shishkin_mesh(16, 1e-3)
    with pytest.raises(spp.SppError) as e:
        spp.Batch1D([16, 15], [1e-3, 1e-3], np.concatenate([x, x]), np.ones(29), np.ones(29))
    assert e.value.code == -1
    xb = np.concatenate([x, x]); xb[20] += 1e-3
    with pytest.raises(spp.SppError) as e:
        spp.Batch1D([16, 16], [1e-3, 1e-3], xb, np.ones(30), np.ones(30))
    assert e.value.code == -2 and "problem 1" in str(e.value)
    c = np.ones(30); c[17] = -1.0
    with pytest.raises(spp.SppError) as e:
        spp.Batch1D([16, 16], [1e-3, 1e-3], np.concatenate([x, x]), c, np.ones(30))
    assert e.value.code == -3 and "problem 1" in str(e.value)


def test_batch_max_iters_cap_not_converged():
    Ns = [512, 512]
    eps = [1e-2, 1e-6]
    xs, cs, rs, fs = build_batch(Ns, eps)
    o = spp.spp_default_options(1)
    o.max_iters = 2
    B = spp.Batch1D(Ns, eps, np.concatenate(xs), dev(np.concatenate(cs)), dev(np.concatenate(rs)), options=o)
    res = B.solve(dev(np.concatenate(fs)))
    assert res.status == spp.SPP_NOT_CONVERGED and list(res.iters) == [2, 2]
    for p in range(2):
        orc = oracle_solve(Ns[p], eps[p], cs[p], rs[p], fs[p], o)
        assert orc["iters"] == 2 and not orc["converged"]
        assert rel(res.u.cpu().numpy()[p * 511:(p + 1) * 511], orc["u"]) <= 1e-9

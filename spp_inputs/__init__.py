"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This module holds the WORKLOAD definitions only -- coefficient functions, right-hand sides,
manufactured solutions and the counter-based random generator -- sampled at mesh nodes that
the caller supplies.  It contains none of the method's arithmetic (no mesh formula, no
stencil, no preconditioner).  Both sides build their own Shishkin mesh (oracle.mesh and
spp_shishkin_mesh in the C ABI; tests assert they agree bit for bit) and pass its node
coordinates here.

Configurations (BASELINE.json ``configs``, B:7-11):
  cfg1  1D  -eps u'' - u' + u = 1 + x,            eps=1e-4, N=256,  rtol 1e-10
  cfg2  2D  c=(1,1), r=1, f from u* = g(x)g(y),    eps=1e-2, N=128,  rtol 1e-10
  cfg3  2D  c=(1+x^2, 1+y^2), r=1+xy, f=e^{x+y},   eps=1e-6, N=1024, rtol 1e-8
  cfg4  2D  c=(1.5+0.5 sin pi x, 1.5+0.5 cos pi y), r=2, f=1+0.1 U(-1,1) seed 0,
            eps=1e-8, N=4096, rtol 1e-8
  cfg5  2D  c=(1,2), r=1, f=1+0.1 U(-1,1) seed 1,  N=8192, eps in {1e-2..1e-10}, rtol 1e-8
  cfg1-batch  many independent 1D problems: see batch1d_params/sample_batch1d
Paper workloads (pins):
  ex1d  eq:1D example:   c = 2 + sin 5x, r = 1, f = 4 e^{-x}, C_lower = 0.99
  exp2d eq:exponential_MMS: c = (2,3), r = 1, f = L u*
  par2d eq:parabolic_MMS: c = (1,0), r = 1, f = L u*: one parabolic layer along
        y = 0 (transition tau_y = sigma sqrt(eps) ln N, eq:tau parabolic: the y mesh is
        built with eps_y = sqrt(eps), beta_y = 1) and one exponential layer along x = 0
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

# ------------------------------------------------------------------ counter-based RNG
_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def splitmix_uniform(seed: int, idx: np.ndarray) -> np.ndarray:
    """U in [0,1): top 53 bits of the SplitMix64 finaliser of key = seed*C1 + idx*C2 + C3
    (SURVEY A14).  Counter-based, so any shard regenerates its own slice."""
    idx = np.asarray(idx, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = (np.uint64(seed) * np.uint64(0xD1B54A32D192ED03)
             + idx * np.uint64(0x9E3779B97F4A7C15) + np.uint64(0x2545F4914F6CDD1D))
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return (z >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)


# ------------------------------------------------------------------ configurations
@dataclass
class Config:
    name: str
    dim: int
    N: int
    eps: float
    tol: float
    sigma: float = 2.0
    beta_x: float = 1.0
    beta_y: float = 1.0
    weighted: int = 1        # Jacobi-weighted residual (reading R11)
    eps_y: float | None = None   # layer scale of the y mesh (None: eps); sqrt(eps) for par2d
    stop_abs: int = 0
    seed: int = 0
    kind: str = ""
    extra: dict = field(default_factory=dict)

    @property
    def unknowns(self) -> int:
        return (self.N - 1) ** self.dim


def config(name: str, N: int | None = None, eps: float | None = None) -> Config:
    """BASELINE configs (optionally at another N / eps, e.g. a proxy size for tests)."""
    base = {
        "cfg1": Config("cfg1", 1, 256, 1e-4, 1e-10, kind="cfg1"),
        "cfg2": Config("cfg2", 2, 128, 1e-2, 1e-10, kind="cfg2"),
        "cfg3": Config("cfg3", 2, 1024, 1e-6, 1e-8, kind="cfg3"),
        "cfg4": Config("cfg4", 2, 4096, 1e-8, 1e-8, kind="cfg4", seed=0),
        "cfg5": Config("cfg5", 2, 8192, 1e-8, 1e-8, kind="cfg5", seed=1),
        # paper workloads
        "ex1d": Config("ex1d", 1, 128, 1e-8, 1.0, sigma=2.0, beta_x=0.99, kind="ex1d"),
        "exp2d": Config("exp2d", 2, 128, 1e-6, 1.0, sigma=2.5, beta_x=1.99, beta_y=2.99,
                        weighted=0, stop_abs=1, kind="exp2d"),
        "par2d": Config("par2d", 2, 128, 1e-6, 1.0, sigma=2.5, beta_x=0.99, beta_y=1.0,
                        weighted=0, stop_abs=1, kind="par2d"),
    }[name]
    if N is not None:
        base.N = N
    if eps is not None:
        base.eps = eps
    if name in ("exp2d", "par2d"):
        # paper 2D stop ||R||_2 <= 10 N^{-1} ln N: a workload parameter
        base.tol = 10.0 * np.log(base.N) / base.N
    if name == "par2d":
        base.eps_y = float(np.sqrt(base.eps))
    if name == "ex1d":
        base.tol = np.log(base.N) / base.N          # K = 1
    return base


def _grid(x, y):
    X, Y = np.meshgrid(np.asarray(x)[1:-1], np.asarray(y)[1:-1], indexing="xy")
    return X, Y            # shape (N-1, N-1), [j-1, i-1]


def _g_cfg2(s, eps):
    """cfg2 factor (B:8, corrected per DESIGN.md reading R13):
    g(s) = s - (1 - e^{-s/eps}) / (1 - e^{-1/eps});  exp underflow gives exactly 0."""
    Q = -np.expm1(-1.0 / eps)
    return s - (-np.expm1(-s / eps)) / Q


def _par_factors(X, Y, e):
    """eq:parabolic_MMS factors: g(x) = cos(pi x/2) - (e^{-x/eps} - e^{-1/eps})/(1 - e^{-1/eps}),
    h(y) = (1 - e^{-y/sqrt eps})/(1 - e^{-1/sqrt eps}) - y^{5/2}."""
    Q = -np.expm1(-1.0 / e)
    s = np.sqrt(e)
    R = -np.expm1(-1.0 / s)
    g = np.cos(np.pi * X / 2) - (np.exp(-X / e) - np.exp(-1.0 / e)) / Q
    h = -np.expm1(-Y / s) / R - Y ** 2.5
    return g, h, R, s


def exact_solution(cfg: Config, x, y=None):
    """Manufactured solution u* at interior nodes (cfg2, exp2d, par2d)."""
    if cfg.kind == "cfg2":
        X, Y = _grid(x, y)
        return _g_cfg2(X, cfg.eps) * _g_cfg2(Y, cfg.eps)
    if cfg.kind == "exp2d":
        X, Y = _grid(x, y)
        e = cfg.eps
        return (np.cos(np.pi * X / 2) * (-np.expm1(-2 * X / e)) * (1 - Y) ** 3
                * (-np.expm1(-3 * Y / e)))
    if cfg.kind == "par2d":
        X, Y = _grid(x, y)
        g, h, _, _ = _par_factors(X, Y, cfg.eps)
        return g * h
    raise KeyError(cfg.kind)


def sample_1d(cfg: Config, x):
    """(c, r, f) at interior nodes x_1..x_{N-1}."""
    xi = np.asarray(x, dtype=np.float64)[1:-1]
    if cfg.kind == "cfg1":          # B:7: -eps u'' - u' + u = 1 + x
        return np.ones_like(xi), np.ones_like(xi), 1.0 + xi
    if cfg.kind == "ex1d":          # eq:1D example
        return 2.0 + np.sin(5.0 * xi), np.ones_like(xi), 4.0 * np.exp(-xi)
    raise KeyError(cfg.kind)


def batch1d_params(nprob: int, seed: int = 7, Ns=(256,), eps_range=(1e-8, 1e-2)):
    """(N_p, eps_p) of a batch of 1D problems: N cycles through Ns, eps log-uniform in
    eps_range (counter-based draws, stream 2*p)."""
    p = np.arange(nprob, dtype=np.uint64)
    u = splitmix_uniform(seed, 2 * p)
    lo, hi = np.log10(eps_range[0]), np.log10(eps_range[1])
    eps = 10.0 ** (lo + (hi - lo) * u)
    N = np.array([Ns[k % len(Ns)] for k in range(nprob)], dtype=np.int32)
    return N, eps


def sample_batch1d(p: int, x, seed: int = 7):
    """(c, r, f) of batch problem p at interior nodes: c = 2 + sin(5x + 2 pi U_p) (>= 1, so
    C_lower = 1), r = 1 + U'_p, f = 1 + x + 0.1 U(-1,1) per node (seed stream p)."""
    xi = np.asarray(x, dtype=np.float64)[1:-1]
    u2 = splitmix_uniform(seed, np.array([2 * p + 1], dtype=np.uint64))[0]
    u3 = splitmix_uniform(seed + 1, np.array([p], dtype=np.uint64))[0]
    noise = 2.0 * splitmix_uniform(seed + 1000 + p, np.arange(xi.size, dtype=np.uint64)) - 1.0
    return 2.0 + np.sin(5.0 * xi + 2.0 * np.pi * u2), (1.0 + u3) * np.ones_like(xi), 1.0 + xi + 0.1 * noise


def sample_2d(cfg: Config, x, y):
    """(c1, c2, r, f) at interior nodes, shape (N-1, N-1) indexed [j-1, i-1]."""
    X, Y = _grid(x, y)
    N, e = cfg.N, cfg.eps
    one = np.ones_like(X)
    if cfg.kind == "cfg2":
        gx, gy = _g_cfg2(X, e), _g_cfg2(Y, e)
        # -eps g'' - g' = -1 identically, so L(g(x)g(y)) = g g - g(x) - g(y)  (c=(1,1), r=1)
        f = gx * gy - gx - gy
        return one, one.copy(), one.copy(), f
    if cfg.kind == "cfg3":          # B:9
        return 1 + X ** 2, 1 + Y ** 2, 1 + X * Y, np.exp(X + Y)
    if cfg.kind in ("cfg4", "cfg5"):
        m = N - 1
        idx = np.arange(m * m, dtype=np.uint64).reshape(m, m)   # (j-1)(N-1)+(i-1)
        f = 1.0 + 0.1 * (2.0 * splitmix_uniform(cfg.seed, idx) - 1.0)
        if cfg.kind == "cfg4":      # B:10
            return 1.5 + 0.5 * np.sin(np.pi * X), 1.5 + 0.5 * np.cos(np.pi * Y), 2.0 * one, f
        return one, 2.0 * one, one.copy(), f   # cfg5, B:11
    if cfg.kind == "exp2d":
        # u = C(x)E(x) P(y)F(y), C = cos(pi x/2), E = 1-e^{-2x/eps}, P = (1-y)^3,
        # F = 1-e^{-3y/eps}; the layer factors satisfy -eps E'' - 2E' = 0 and
        # -eps F'' - 3F' = 0 exactly, so f = gy*A1 + gx*A2 + gx*gy with the O(1) forms below.
        C = np.cos(np.pi * X / 2)
        C1 = -(np.pi / 2) * np.sin(np.pi * X / 2)
        C2 = -(np.pi / 2) ** 2 * C
        e1 = np.exp(-2 * X / e)
        E = -np.expm1(-2 * X / e)
        P = (1 - Y) ** 3
        P1 = -3 * (1 - Y) ** 2
        P2 = 6 * (1 - Y)
        e2 = np.exp(-3 * Y / e)
        F = -np.expm1(-3 * Y / e)
        gx, gy = C * E, P * F
        A1 = -e * C2 * E - 4 * C1 * e1 - 2 * C1 * E
        A2 = -e * P2 * F - 6 * P1 * e2 - 3 * P1 * F
        f = gy * A1 + gx * A2 + gx * gy
        return 2.0 * one, 3.0 * one, one.copy(), f
    if cfg.kind == "par2d":
        # -eps Lap u - u_x + u with u = g(x) h(y): the layer parts of g satisfy -eps g'' - g' = 0
        # exactly, so -eps g'' - g' = eps (pi/2)^2 cos(pi x/2) + (pi/2) sin(pi x/2); and
        # -eps h'' = e^{-y/sqrt eps}/R + (15/4) eps y^{1/2}
        g, h, R, s = _par_factors(X, Y, e)
        Ax = e * (np.pi / 2) ** 2 * np.cos(np.pi * X / 2) + (np.pi / 2) * np.sin(np.pi * X / 2)
        By = np.exp(-Y / s) / R + 3.75 * e * np.sqrt(Y)
        f = Ax * h + g * By + g * h
        return one, 0.0 * one, one.copy(), f
    raise KeyError(cfg.kind)


def random_field(seed: int, shape) -> np.ndarray:
    """Generic seeded test vector in [-1, 1) (counter-based)."""
    n = int(np.prod(shape))
    return (2.0 * splitmix_uniform(seed, np.arange(n, dtype=np.uint64)) - 1.0).reshape(shape)

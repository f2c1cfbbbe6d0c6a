"""CPU oracle for arXiv 2108.13468 (ctypes wrapper around ``spp_oracle.c``).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this package.  The
product path (``paper_2108_13468_b200``) never imports it, and the two share no code.

Array convention: 2D grid functions are numpy arrays of shape (N-1, N-1) indexed
``[j-1, i-1]`` (row = y index), i.e. the flat index (j-1)(N-1)+(i-1) of SURVEY 8(b).
Corner-block arrays are (N/2, N/2) indexed the same way.

Functions whose result has no independent pin are marked "parity unpinned" in their
docstring (none at present).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_SRC = _HERE / "spp_oracle.c"
_LIB = _HERE / "liboracle.so"

_dp = ctypes.POINTER(ctypes.c_double)
_ip = ctypes.POINTER(ctypes.c_int)


def build(force: bool = False) -> Path:
    """Compile the oracle with gcc -O2 -ffp-contract=off (plain, no FMA contraction)."""
    if force or not _LIB.exists() or _LIB.stat().st_mtime < _SRC.stat().st_mtime:
        tmp = _LIB.with_suffix(f".so.tmp{os.getpid()}")
        subprocess.check_call(
            ["gcc", "-std=c11", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared",
             "-Wall", "-o", str(tmp), str(_SRC), "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(str(_LIB))
        L.orc_mesh.argtypes = [ctypes.c_int, ctypes.c_double, ctypes.c_double, ctypes.c_double, _dp]
        L.orc_mesh_bs.argtypes = [ctypes.c_int, ctypes.c_double, ctypes.c_double, ctypes.c_double, _dp]
        L.orc_thomas.argtypes = [ctypes.c_int, _dp, _dp, _dp, _dp, _dp]
        L.orc1_coef.argtypes = [ctypes.c_int, ctypes.c_double, _dp, _dp, _dp, _dp, _dp, _dp]
        L.orc1_matvec.argtypes = [ctypes.c_int, _dp, _dp, _dp, _dp, _dp]
        L.orc1_direct.argtypes = [ctypes.c_int, _dp, _dp, _dp, _dp, _dp, _dp]
        L.orc1_precond.argtypes = [ctypes.c_int, _dp, _dp, _dp, _dp, _dp]
        L.orc1_solve.argtypes = [ctypes.c_int, ctypes.c_double, _dp, _dp, _dp, _dp, ctypes.c_int,
                                 ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.c_int,
                                 ctypes.c_int, _dp, _dp, ctypes.c_int, _ip, _dp]
        L.orc2_create.argtypes = [ctypes.c_int, ctypes.c_double, _dp, _dp, _dp, _dp, _dp,
                                  ctypes.c_double, ctypes.c_int, ctypes.c_int]
        L.orc2_create.restype = ctypes.c_void_p
        L.orc2_destroy.argtypes = [ctypes.c_void_p]
        L.orc2_solve.argtypes = [ctypes.c_void_p, _dp, _dp, ctypes.c_int, ctypes.c_int,
                                 ctypes.c_double, ctypes.c_int, ctypes.c_int, _dp, ctypes.c_int,
                                 _ip, _dp]
        L.orc2_solve_r.argtypes = [ctypes.c_void_p, _dp, _dp, ctypes.c_int, ctypes.c_int,
                                   ctypes.c_double, ctypes.c_int, ctypes.c_int, ctypes.c_int, _dp,
                                   ctypes.c_int, _ip, _dp]
        L.orc2_levels.argtypes = [ctypes.c_void_p]
        L.orc2_level_n.argtypes = [ctypes.c_void_p, ctypes.c_int]
        L.orc2_get_coef.argtypes = [ctypes.c_void_p, _dp, _dp, _dp, _dp, _dp]
        L.orc2_get_level_coef.argtypes = [ctypes.c_void_p, ctypes.c_int, _dp, _dp, _dp, _dp, _dp,
                                          _dp, _dp]
        L.orc2_matvec.argtypes = [ctypes.c_void_p, _dp, _dp]
        L.orc2_precond.argtypes = [ctypes.c_void_p, _dp, _dp]
        L.orc2_stage_I.argtypes = [ctypes.c_void_p, _dp, _dp]
        L.orc2_stage_Y.argtypes = [ctypes.c_void_p, _dp, _dp]
        L.orc2_stage_X.argtypes = [ctypes.c_void_p, _dp, _dp]
        L.orc2_corner_rhs.argtypes = [ctypes.c_void_p, _dp, _dp, _dp]
        L.orc2_corner_solve_ext.argtypes = [ctypes.c_void_p, _dp, _dp, _ip]
        L.orc2_gs_sweep.argtypes = [ctypes.c_void_p, ctypes.c_int, _dp, _dp]
        L.orc2_vcycle.argtypes = [ctypes.c_void_p, ctypes.c_int, _dp, _dp]
        L.orc2_level_residual.argtypes = [ctypes.c_void_p, ctypes.c_int, _dp, _dp, _dp]
        L.orc2_restrict.argtypes = [ctypes.c_void_p, ctypes.c_int, _dp, _dp]
        L.orc2_prolong_add.argtypes = [ctypes.c_void_p, ctypes.c_int, _dp, _dp]
        L.orc2_set_mg.argtypes = [ctypes.c_void_p, ctypes.c_double, ctypes.c_int, ctypes.c_int]
        L.orc2_cycle_log.argtypes = [ctypes.c_void_p, _ip, ctypes.c_int]
        L.orc2_direct.argtypes = [ctypes.c_void_p, _dp, _dp, ctypes.c_int]
        for nm in ("orc2_par", "orc2_plevels"):
            getattr(L, nm).argtypes = [ctypes.c_void_p]
        L.orc2_plevel_nx.argtypes = [ctypes.c_void_p, ctypes.c_int]
        L.orc2_plevel_stencil.argtypes = [ctypes.c_void_p, ctypes.c_int, _dp]
        L.orc2_pgs.argtypes = [ctypes.c_void_p, ctypes.c_int, _dp, _dp]
        L.orc2_pvcycle.argtypes = [ctypes.c_void_p, ctypes.c_int, _dp, _dp]
        L.orc2_presidual.argtypes = [ctypes.c_void_p, ctypes.c_int, _dp, _dp, _dp]
        L.orc2_prestrict.argtypes = [ctypes.c_void_p, ctypes.c_int, _dp, _dp]
        L.orc2_pprolong_add.argtypes = [ctypes.c_void_p, ctypes.c_int, _dp, _dp]
        _lib = L
    return _lib


def _p(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_dp)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


# ------------------------------------------------------------------------------ mesh
def mesh(N: int, eps: float, sigma: float = 2.0, beta: float = 1.0) -> np.ndarray:
    """Shishkin mesh, eq:tau 1D / eq:tau exponential."""
    x = np.zeros(N + 1)
    rc = lib().orc_mesh(N, eps, sigma, beta, _p(x))
    if rc != 0:
        raise ValueError(f"orc_mesh rc={rc}")
    return x


def mesh_bs(N: int, eps: float, sigma: float = 2.0, beta: float = 1.0) -> np.ndarray:
    """Bakhvalov-Shishkin graded mesh (NEXT-4, reading R21)."""
    x = np.zeros(N + 1)
    rc = lib().orc_mesh_bs(N, eps, sigma, beta, _p(x))
    if rc != 0:
        raise ValueError(f"orc_mesh_bs rc={rc}")
    return x


def thomas(lo, di, up, rhs):
    lo, di, up, rhs = map(_f64, (lo, di, up, rhs))
    x = np.zeros_like(rhs)
    rc = lib().orc_thomas(len(di), _p(lo), _p(di), _p(up), _p(rhs), _p(x))
    if rc != 0:
        raise ArithmeticError(f"thomas rc={rc}")
    return x


# ------------------------------------------------------------------------------ 1D
def coef1d(N, eps, x, c, r):
    """Difference-form coefficients of eq:stencil_1d: (aW, aE, D)."""
    x, c, r = map(_f64, (x, c, r))
    aW, aE, D = (np.zeros(N - 1) for _ in range(3))
    lib().orc1_coef(N, eps, _p(x), _p(c), _p(r), _p(aW), _p(aE), _p(D))
    return aW, aE, D


def matvec1d(N, eps, x, c, r, u):
    aW, aE, D = coef1d(N, eps, x, c, r)
    u = _f64(u)
    y = np.zeros(N - 1)
    lib().orc1_matvec(N, _p(aW), _p(aE), _p(_f64(r)), _p(u), _p(y))
    return y


def direct1d(N, eps, x, c, r, f):
    aW, aE, D = coef1d(N, eps, x, c, r)
    u = np.zeros(N - 1)
    rc = lib().orc1_direct(N, _p(aW), _p(aE), _p(D), _p(_f64(r)), _p(_f64(f)), _p(u))
    if rc != 0:
        raise ArithmeticError(rc)
    return u


def precond1d(N, eps, x, c, r, q):
    aW, aE, D = coef1d(N, eps, x, c, r)
    z = np.zeros(N - 1)
    rc = lib().orc1_precond(N, _p(aW), _p(aE), _p(D), _p(_f64(q)), _p(z))
    if rc != 0:
        raise ArithmeticError(rc)
    return z


def solve1d(N, eps, x, c, r, f, *, side=0, weighted=1, stop_abs=0, tol=1e-10, maxit=200,
            fixed_iters=0):
    """1D GMRES: side=0 right/flexible (BASELINE, Jacobi-weighted by default), side=1 left
    with the true inf-norm residual stop of P:812 (paper mode)."""
    x, c, r, f = map(_f64, (x, c, r, f))
    u = np.zeros(N - 1)
    hist = np.zeros(maxit + 2)
    oi = (ctypes.c_int * 8)()
    od = (ctypes.c_double * 4)()
    rc = lib().orc1_solve(N, eps, _p(x), _p(c), _p(r), _p(f), side, weighted, stop_abs, tol, maxit,
                          fixed_iters, _p(u), _p(hist), len(hist), oi, od)
    if rc < 0:
        raise RuntimeError(f"orc1_solve rc={rc}")
    it = oi[0]
    return dict(u=u, hist=hist[: it + 1].copy(), iters=it, converged=bool(oi[1]), res0=od[0],
                res_final=od[1], status=rc)


# ------------------------------------------------------------------------------ 2D
class Oracle2D:
    """2D two-exponential-layer problem, block preconditioner + corner MG + FGMRES."""

    def __init__(self, N, eps, x, y, c1, c2, r, mg_red=1e-3, mg_cap=20, mg_fixed=0):
        self.N, self.n, self.m, self.eps = N, N // 2, N - 1, eps
        arrs = [_f64(a) for a in (x, y, c1, c2, r)]
        self._keep = arrs
        self.h = lib().orc2_create(N, eps, *[_p(a) for a in arrs], mg_red, mg_cap, mg_fixed)
        if not self.h:
            raise ValueError("orc2_create failed (N must be even, N/2 a power of two >= 4)")

    def close(self):
        if self.h:
            lib().orc2_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _g(self, a=None):
        return np.zeros((self.m, self.m)) if a is None else _f64(a).reshape(self.m, self.m)

    def set_mg(self, red=1e-3, cap=20, fixed=0):
        lib().orc2_set_mg(self.h, red, cap, fixed)

    @property
    def levels(self):
        return lib().orc2_levels(self.h)

    # --- parabolic-layer corner (c2 = 0): semi-coarsening Galerkin levels, nine-point (NEXT-2)
    @property
    def parabolic(self):
        return bool(lib().orc2_par(self.h))

    @property
    def plevels(self):
        return lib().orc2_plevels(self.h)

    def plevel_shape(self, l):
        return self.n, lib().orc2_plevel_nx(self.h, l)      # (rows ny, columns nx)

    def _pv(self, l, a=None):
        ny, nx = self.plevel_shape(l)
        return np.zeros((ny, nx)) if a is None else _f64(a).reshape(ny, nx)

    def plevel_stencil(self, l):
        ny, nx = self.plevel_shape(l)
        a = np.zeros((ny, nx, 9))
        lib().orc2_plevel_stencil(self.h, l, _p(a))
        return a                                             # [j-1, i-1, (dj+1)*3 + (di+1)]

    def pgs(self, l, b, e):
        b, e = self._pv(l, b), self._pv(l, e).copy()
        lib().orc2_pgs(self.h, l, _p(b), _p(e))
        return e

    def pvcycle(self, l, b):
        b, e = self._pv(l, b), self._pv(l)
        lib().orc2_pvcycle(self.h, l, _p(b), _p(e))
        return e

    def presidual(self, l, b, e):
        b, e, r = self._pv(l, b), self._pv(l, e), self._pv(l)
        lib().orc2_presidual(self.h, l, _p(b), _p(e), _p(r))
        return r

    def prestrict(self, l, r):
        r, bc = self._pv(l, r), self._pv(l + 1)
        lib().orc2_prestrict(self.h, l, _p(r), _p(bc))
        return bc

    def pprolong_add(self, l, ec, e):
        ec, e = self._pv(l + 1, ec), self._pv(l, e).copy()
        lib().orc2_pprolong_add(self.h, l, _p(ec), _p(e))
        return e

    def level_n(self, l):
        return lib().orc2_level_n(self.h, l)

    def coef(self):
        N, m = self.N, self.m
        aW, aS = np.zeros(N + 1), np.zeros(N + 1)
        aE, aN, D = (np.zeros((m, m)) for _ in range(3))
        lib().orc2_get_coef(self.h, _p(aW), _p(aS), _p(aE), _p(aN), _p(D))
        return dict(aW=aW, aS=aS, aE=aE, aN=aN, D=D)

    def level_coef(self, l):
        nl = self.level_n(l)
        aW, aS, hb, kb = (np.zeros(nl + 2) for _ in range(4))
        aE, aN, D = (np.zeros((nl, nl)) for _ in range(3))
        lib().orc2_get_level_coef(self.h, l, _p(aW), _p(aS), _p(aE), _p(aN), _p(D), _p(hb), _p(kb))
        return dict(aW=aW, aS=aS, aE=aE, aN=aN, D=D, hb=hb, kb=kb, n=nl)

    def matvec(self, u):
        u = self._g(u)
        y = self._g()
        lib().orc2_matvec(self.h, _p(u), _p(y))
        return y

    def precond(self, q):
        q = self._g(q)
        z = self._g()
        rc = lib().orc2_precond(self.h, _p(q), _p(z))
        if rc != 0:
            raise RuntimeError(rc)
        return z

    def stage_I(self, q, z=None):
        q = self._g(q)
        z = self._g(z).copy()
        lib().orc2_stage_I(self.h, _p(q), _p(z))
        return z

    def stage_Y(self, q, z):
        q, z = self._g(q), self._g(z).copy()
        lib().orc2_stage_Y(self.h, _p(q), _p(z))
        return z

    def stage_X(self, q, z):
        q, z = self._g(q), self._g(z).copy()
        lib().orc2_stage_X(self.h, _p(q), _p(z))
        return z

    def corner_rhs(self, q, z):
        q, z = self._g(q), self._g(z)
        b = np.zeros((self.n, self.n))
        lib().orc2_corner_rhs(self.h, _p(q), _p(z), _p(b))
        return b

    def corner_solve(self, bC):
        bC = _f64(bC).reshape(self.n, self.n)
        z = np.zeros_like(bC)
        cap = ctypes.c_int(0)
        cyc = lib().orc2_corner_solve_ext(self.h, _p(bC), _p(z), ctypes.byref(cap))
        return z, cyc, bool(cap.value)

    def _lv(self, l, a=None):
        nl = self.level_n(l)
        return np.zeros((nl, nl)) if a is None else _f64(a).reshape(nl, nl)

    def gs_sweep(self, l, b, e):
        b, e = self._lv(l, b), self._lv(l, e).copy()
        lib().orc2_gs_sweep(self.h, l, _p(b), _p(e))
        return e

    def vcycle(self, l, b):
        b = self._lv(l, b)
        e = self._lv(l)
        lib().orc2_vcycle(self.h, l, _p(b), _p(e))
        return e

    def level_residual(self, l, b, e):
        b, e = self._lv(l, b), self._lv(l, e)
        rho = self._lv(l)
        lib().orc2_level_residual(self.h, l, _p(b), _p(e), _p(rho))
        return rho

    def restrict(self, l, rho):
        rho = self._lv(l, rho)
        bc = self._lv(l + 1)
        lib().orc2_restrict(self.h, l, _p(rho), _p(bc))
        return bc

    def prolong_add(self, l, ec, e):
        ec, e = self._lv(l + 1, ec), self._lv(l, e).copy()
        lib().orc2_prolong_add(self.h, l, _p(ec), _p(e))
        return e

    def cycle_log(self):
        buf = (ctypes.c_int * 4096)()
        k = lib().orc2_cycle_log(self.h, buf, 4096)
        return list(buf[: min(k, 4096)])

    def direct(self, f, refine=8):
        f = self._g(f)
        u = self._g()
        rc = lib().orc2_direct(self.h, _p(f), _p(u), refine)
        if rc != 0:
            raise RuntimeError(rc)
        return u

    def solve(self, f, *, weighted=1, stop_abs=0, tol=1e-8, maxit=200, fixed_iters=0, restart=0):
        """FGMRES (restart = 0, the paper) or FGMRES(restart) (reading R23)"""
        f = self._g(f)
        u = self._g()
        hist = np.zeros(maxit + 2)
        oi = (ctypes.c_int * 8)()
        od = (ctypes.c_double * 4)()
        rc = lib().orc2_solve_r(self.h, _p(f), _p(u), weighted, stop_abs, tol, maxit, fixed_iters,
                                restart, _p(hist), len(hist), oi, od)
        if rc < 0:
            raise RuntimeError(f"orc2_solve rc={rc}")
        it = oi[0]
        return dict(u=u, hist=hist[: it + 1].copy(), iters=it, converged=bool(oi[1]),
                    mg_cycles_total=oi[2], mg_cycles_min=oi[3], mg_cycles_max=oi[4],
                    mg_cap_hits=oi[5], applies=oi[6], res0=od[0], res_final=od[1], status=rc,
                    cycle_log=self.cycle_log())

"""Python binding of the B200 solver C ABI (include/spp.h) -- argument marshalling only.

Every step of the hot path runs in the sm_100a kernels of ``lib/libspp.so``; this module only
converts arguments (numpy arrays for host memory, torch CUDA tensors for device memory) and
calls the ABI functions of the same names.  There is no CPU path: if the shared library is
missing this import fails, and if no CUDA device is present ``spp_create`` fails.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass
from pathlib import Path

import numpy as np

_PKG = Path(__file__).resolve().parent
LIB_PATH = _PKG / "lib" / "libspp.so"

SPP_OK, SPP_NOT_CONVERGED = 0, 1
(SPP_E_ARG, SPP_E_MESH, SPP_E_COEF, SPP_E_PIVOT, SPP_E_MG_CAP, SPP_E_CUDA, SPP_E_NCCL, SPP_E_NOMEM, SPP_E_STATE,
 SPP_E_NONFINITE) = range(-1, -11, -1)
SPP_HOST, SPP_DEVICE = 0, 1
SPP_STOP_REL_JACOBI, SPP_STOP_REL_L2, SPP_STOP_ABS_L2, SPP_STOP_ABS_MAX = 0, 1, 2, 3
SPP_RIGHT_FLEXIBLE, SPP_LEFT = 0, 1
STAGES = dict(MATVEC=0, MII=1, MYY=2, MXX=3, CORNER_RHS=4, GS_SWEEP=5, VCYCLE=6, CORNER_SOLVE=7,
              PRECOND=8, RESTRICT=9, PROLONG_ADD=10, LEVEL_RESIDUAL=11, MII_JACOBI=12, POST_SMOOTH=13,
              RESID_RESTRICT=14, PRE_RESTRICT=15)
PROF_CLASSES = 12


class spp_problem(ctypes.Structure):
    _fields_ = [("dim", ctypes.c_int32), ("n", ctypes.c_int32), ("eps", ctypes.c_double),
                ("x", ctypes.c_void_p), ("y", ctypes.c_void_p), ("c1", ctypes.c_void_p),
                ("c2", ctypes.c_void_p), ("r", ctypes.c_void_p), ("mem", ctypes.c_int)]


class spp_options(ctypes.Structure):
    _fields_ = [("side", ctypes.c_int), ("stop", ctypes.c_int), ("tol", ctypes.c_double),
                ("max_iters", ctypes.c_int32), ("restart", ctypes.c_int32),
                ("mg_reduction", ctypes.c_double), ("mg_max_cycles", ctypes.c_int32),
                ("mg_fixed_cycles", ctypes.c_int32), ("mg_coarsest", ctypes.c_int32),
                ("fixed_iters", ctypes.c_int32), ("mg_strict", ctypes.c_int32),
                ("reserved", ctypes.c_int32 * 7)]


class spp_stats(ctypes.Structure):
    _fields_ = [("iters", ctypes.c_int32), ("converged", ctypes.c_int32),
                ("mg_cycles_total", ctypes.c_int32), ("mg_cycles_min", ctypes.c_int32),
                ("mg_cycles_max", ctypes.c_int32), ("mg_cap_hits", ctypes.c_int32),
                ("applies", ctypes.c_int32), ("kernel_launches", ctypes.c_int32),
                ("res0", ctypes.c_double), ("res_final", ctypes.c_double),
                ("true_res_l2_rel", ctypes.c_double), ("true_res_jacobi_rel", ctypes.c_double),
                ("setup_s", ctypes.c_double), ("solve_s", ctypes.c_double)]

    def asdict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


# names declared in include/spp.h (checked against the header by tests/test_abi.py)
ABI_FUNCTIONS = ["spp_default_options", "spp_shishkin_mesh", "spp_bakhvalov_mesh", "spp_create", "spp_setup",
                 "spp_solve", "spp_apply_stage", "spp_kernel_launches", "spp_mg_levels", "spp_mg_level_n",
                 "spp_profile_enable", "spp_profile_reset", "spp_profile_get", "spp_profile_name",
                 "spp_destroy", "spp_last_error", "spp_version",
                 "spp_batch1d_create", "spp_batch1d_setup", "spp_batch1d_solve", "spp_batch1d_nprob", "spp_batch1d_launches",
                 "spp_batch1d_last_error", "spp_batch1d_destroy",
                 "spp_strip_partition", "spp_create_strips", "spp_create_dist", "spp_nccl_unique_id",
                 "spp_nccl_comm_create", "spp_nccl_comm_destroy", "spp_dist_info", "spp_dist_plan"]

if not LIB_PATH.exists():
    raise ImportError(f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                      f"g.build()'` (there is no CPU fallback)")
_lib = ctypes.CDLL(str(LIB_PATH))
_vp, _dp = ctypes.c_void_p, ctypes.POINTER(ctypes.c_double)
_lib.spp_default_options.argtypes = [ctypes.c_int32, ctypes.POINTER(spp_options)]
_lib.spp_default_options.restype = None
_lib.spp_shishkin_mesh.argtypes = [ctypes.c_int32, ctypes.c_double, ctypes.c_double, ctypes.c_double, _dp]
_lib.spp_bakhvalov_mesh.argtypes = [ctypes.c_int32, ctypes.c_double, ctypes.c_double, ctypes.c_double, _dp]
_lib.spp_create.argtypes = [ctypes.POINTER(spp_problem), ctypes.POINTER(spp_options), _vp, ctypes.POINTER(_vp)]
_lib.spp_setup.argtypes = [_vp, _vp, _vp, _vp, ctypes.c_int]
_lib.spp_solve.argtypes = [_vp, _vp, _vp, ctypes.c_int, _dp, ctypes.c_int32, ctypes.POINTER(spp_stats)]
_lib.spp_apply_stage.argtypes = [_vp, ctypes.c_int, ctypes.c_int32, _vp, _vp, ctypes.POINTER(ctypes.c_int32)]
_lib.spp_kernel_launches.argtypes = [_vp]
_lib.spp_kernel_launches.restype = ctypes.c_int64
_lib.spp_mg_levels.argtypes = [_vp]
_lib.spp_mg_level_n.argtypes = [_vp, ctypes.c_int32]
_lib.spp_profile_enable.argtypes = [_vp, ctypes.c_int32]
_lib.spp_profile_reset.argtypes = [_vp]
_lib.spp_profile_get.argtypes = [_vp, ctypes.c_int32, ctypes.POINTER(ctypes.c_int64),
                                 ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double)]
_lib.spp_profile_name.argtypes = [ctypes.c_int32]
_lib.spp_profile_name.restype = ctypes.c_char_p
_lib.spp_destroy.argtypes = [_vp]
_lib.spp_destroy.restype = None
_lib.spp_last_error.argtypes = [_vp]
_lib.spp_last_error.restype = ctypes.c_char_p
_lib.spp_version.argtypes = []
_lib.spp_version.restype = ctypes.c_char_p
_ip = ctypes.POINTER(ctypes.c_int32)
_lib.spp_batch1d_create.argtypes = [ctypes.c_int32, _ip, _dp, _dp, _vp, _vp, ctypes.c_int,
                                    ctypes.POINTER(spp_options), _vp, ctypes.POINTER(_vp)]
_lib.spp_batch1d_setup.argtypes = [_vp, _vp, _vp, ctypes.c_int]
_lib.spp_batch1d_solve.argtypes = [_vp, _vp, _vp, ctypes.c_int, _ip, _ip, _dp, ctypes.POINTER(spp_stats)]
_lib.spp_batch1d_nprob.argtypes = [_vp]
_lib.spp_batch1d_launches.argtypes = [_vp]
_lib.spp_batch1d_launches.restype = ctypes.c_int64
_lib.spp_batch1d_last_error.argtypes = [_vp]
_lib.spp_batch1d_last_error.restype = ctypes.c_char_p
_lib.spp_batch1d_destroy.argtypes = [_vp]
_lib.spp_batch1d_destroy.restype = None
_lib.spp_strip_partition.argtypes = [ctypes.c_int32, ctypes.c_int32, _ip]
_lib.spp_create_strips.argtypes = [ctypes.POINTER(spp_problem), ctypes.c_int32, ctypes.POINTER(spp_options), _vp,
                                   ctypes.POINTER(_vp)]
_lib.spp_create_dist.argtypes = [ctypes.POINTER(spp_problem), ctypes.c_int32, ctypes.c_int32, _vp, ctypes.c_int32,
                                 ctypes.c_int32, ctypes.POINTER(spp_options), _vp, ctypes.POINTER(_vp)]
_lib.spp_nccl_unique_id.argtypes = [ctypes.c_char_p]
_lib.spp_nccl_comm_create.argtypes = [ctypes.c_char_p, ctypes.c_int32, ctypes.c_int32, ctypes.POINTER(_vp)]
_lib.spp_nccl_comm_destroy.argtypes = [_vp]
_lib.spp_nccl_comm_destroy.restype = None
_lib.spp_dist_info.argtypes = [_vp, _ip, _ip, ctypes.POINTER(ctypes.c_int64), _dp, ctypes.POINTER(ctypes.c_int64)]
_lib.spp_dist_plan.argtypes = [ctypes.c_int32, ctypes.c_int32, _ip, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                               ctypes.c_int32, ctypes.POINTER(ctypes.c_int64), ctypes.c_int32]


class SppError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"spp error {code}: {msg}")
        self.code = code


class SppArgError(SppError, ValueError, TypeError):
    """An argument the binding rejects before calling the library (sizes, dtypes, residency):
    SPP_E_ARG, as the library would report it."""

    def __init__(self, msg):
        super().__init__(-1, msg)


def _check(rc, ctx=None):
    if rc < 0:
        raise SppError(rc, (_lib.spp_last_error(ctx) or b"").decode())
    return rc


def spp_version() -> str:
    return _lib.spp_version().decode()


def spp_default_options(dim: int) -> spp_options:
    o = spp_options()
    _lib.spp_default_options(dim, ctypes.byref(o))
    return o


def spp_bakhvalov_mesh(n: int, eps: float, sigma: float = 2.0, beta: float = 1.0) -> np.ndarray:
    """Bakhvalov-Shishkin graded mesh (spp.h; NEXT-4)."""
    x = np.zeros(n + 1)
    _check(_lib.spp_bakhvalov_mesh(n, eps, sigma, beta, x.ctypes.data_as(_dp)))
    return x


def spp_strip_partition(n: int, nranks: int) -> np.ndarray:
    """Default row strips (spp.h): rank r owns interior rows J[r] .. J[r+1]-1."""
    j = np.zeros(nranks + 1, np.int32)
    _check(_lib.spp_strip_partition(n, nranks, j.ctypes.data_as(_ip)))
    return j


def spp_dist_plan(n: int, nranks: int, j, d_levels: int, halo: int, warm: int, rank: int = -1) -> np.ndarray:
    """Host-only exchange schedule of one FGMRES iteration (spp.h): rows of
    (step, src, dst, role, slot, soff, doff, width, rows, pitch, 0)."""
    j = np.ascontiguousarray(j, dtype=np.int32)
    cnt = _check(_lib.spp_dist_plan(n, nranks, j.ctypes.data_as(_ip), d_levels, halo, warm, rank, None, 0))
    out = np.zeros((max(cnt, 1), 11), np.int64)
    _lib.spp_dist_plan(n, nranks, j.ctypes.data_as(_ip), d_levels, halo, warm, rank,
                       out.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), cnt)
    return out[:cnt]


def nccl_unique_id() -> bytes:
    _nccl_env()
    buf = ctypes.create_string_buffer(128)
    _check(_lib.spp_nccl_unique_id(buf))
    return buf.raw


def nccl_comm_create(uid: bytes, nranks: int, rank: int):
    _nccl_env()
    h = _vp()
    _check(_lib.spp_nccl_comm_create(uid, nranks, rank, ctypes.byref(h)))
    return h


def nccl_comm_destroy(comm):
    _lib.spp_nccl_comm_destroy(comm)


def _nccl_env():
    """Point the library at the libnccl torch uses (one NCCL per process)."""
    import os
    if os.environ.get("SPP_NCCL_LIB"):
        return
    try:
        import nvidia.nccl
        cand = Path(list(nvidia.nccl.__path__)[0]) / "lib" / "libnccl.so.2"
        if cand.exists():
            os.environ["SPP_NCCL_LIB"] = str(cand)
    except Exception:
        pass


def spp_shishkin_mesh(n: int, eps: float, sigma: float = 2.0, beta: float = 1.0) -> np.ndarray:
    x = np.zeros(n + 1)
    _check(_lib.spp_shishkin_mesh(n, eps, sigma, beta, x.ctypes.data_as(_dp)))
    return x


def _ptr(a):
    """(pointer, mem, keepalive) for a numpy array (host) or a torch CUDA tensor (device)."""
    if a is None:
        return None, None, None
    if isinstance(a, np.ndarray):
        a = np.ascontiguousarray(a, dtype=np.float64)
        return a.ctypes.data, SPP_HOST, a
    # torch tensor
    if a.dtype.__str__() != "torch.float64" or not a.is_contiguous():
        raise TypeError("device arrays must be contiguous torch.float64 tensors")
    return a.data_ptr(), (SPP_DEVICE if a.is_cuda else SPP_HOST), a


def _where(a):
    """Residency key of an array: 'host' or the CUDA device it lives on."""
    if isinstance(a, np.ndarray) or not getattr(a, "is_cuda", False):
        return "host"
    return str(a.device)


def _check_arrays(named, count):
    """Every array must have exactly `count` float64 elements and all must share one residency
    (host, or one CUDA device): the library trusts these sizes and the mem flag (spp.h)."""
    where = None
    for name, a in named:
        if a is None:
            continue
        n = a.size if isinstance(a, np.ndarray) else a.numel()
        if n != count:
            raise SppArgError(f"{name}: {n} elements, expected {count}")
        if str(getattr(a, "dtype", "")) not in ("float64", "torch.float64"):
            raise SppArgError(f"{name}: dtype {a.dtype}, expected float64")
        w = _where(a)
        if where is None:
            where = w
        elif w != where:
            raise SppArgError(f"{name} lives on {w}, the other arrays on {where}: one residency per call")


def _stream_handle(stream):
    if stream is None:
        try:
            import torch
            if torch.cuda.is_available():
                return torch.cuda.current_stream().cuda_stream
        except Exception:
            pass
        return None
    return getattr(stream, "cuda_stream", stream)


@dataclass
class SolveResult:
    u: object
    hist: np.ndarray
    status: int
    stats: dict


class Solver:
    """One spp_ctx.  Coefficients/right-hand sides may be numpy arrays (host) or torch CUDA
    float64 tensors (device), in the compact layout (N-1)^dim, x fastest."""

    def __init__(self, dim, n, eps, x, y, c1, c2, r, options: spp_options | None = None, stream=None, strips=1):
        """strips > 1: the row-strip decomposition (spp_create_strips) on this device."""
        self.dim, self.n, self.eps = dim, n, eps
        self.opt = options if options is not None else spp_default_options(dim)
        self._x = np.ascontiguousarray(x, dtype=np.float64)
        self._y = None if y is None else np.ascontiguousarray(y, dtype=np.float64)
        if self._x.size != n + 1 or (dim == 2 and (self._y is None or self._y.size != n + 1)):
            raise SppArgError(f"mesh coordinates: need {n + 1} values per axis")
        _check_arrays([("c1", c1), ("c2", c2), ("r", r)], (n - 1) ** dim)
        p1, mem, k1 = _ptr(c1)
        p2, _, k2 = _ptr(c2)
        p3, _, k3 = _ptr(r)
        prob = spp_problem(dim, n, eps, self._x.ctypes.data, None if self._y is None else self._y.ctypes.data,
                           p1, p2, p3, mem)
        h = _vp()
        self._stream = _stream_handle(stream)
        if strips > 1:
            rc = _lib.spp_create_strips(ctypes.byref(prob), strips, ctypes.byref(self.opt), self._stream, ctypes.byref(h))
        else:
            rc = _lib.spp_create(ctypes.byref(prob), ctypes.byref(self.opt), self._stream, ctypes.byref(h))
        _check(rc)
        self.h = h
        self._keep = (k1, k2, k3)

    def close(self):
        if getattr(self, "h", None):
            _lib.spp_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def m(self):
        return self.n - 1

    def setup(self, c1, c2, r):
        _check_arrays([("c1", c1), ("c2", c2), ("r", r)], self.m ** self.dim)
        p1, mem, k1 = _ptr(c1)
        p2, _, k2 = _ptr(c2)
        p3, _, k3 = _ptr(r)
        _check(_lib.spp_setup(self.h, p1, p2, p3, mem), self.h)

    def solve(self, f, u=None, hist_cap=256) -> SolveResult:
        pf, mem, kf = _ptr(f)
        if u is None:
            if mem == SPP_HOST:
                u = np.zeros(self.m ** self.dim)
            else:
                import torch
                u = torch.zeros_like(f)
        _check_arrays([("f", f), ("u", u)], self.m ** self.dim)
        pu, memu, ku = _ptr(u)
        if memu != mem:
            raise ValueError("f and u must have the same residency")
        hist = np.zeros(hist_cap)
        st = spp_stats()
        rc = _check(_lib.spp_solve(self.h, pf, pu, mem, hist.ctypes.data_as(_dp), hist_cap, ctypes.byref(st)), self.h)
        d = st.asdict()
        return SolveResult(u=ku if mem == SPP_HOST else u, hist=hist[: d["iters"] + 1].copy(), status=rc, stats=d)

    def apply_stage(self, stage, inp, out, level=0):
        """Test hook: inp/out are torch CUDA float64 tensors (device pointers)."""
        cyc = ctypes.c_int32(0)
        s = STAGES[stage] if isinstance(stage, str) else stage
        _check(_lib.spp_apply_stage(self.h, s, level, inp.data_ptr(), out.data_ptr(), ctypes.byref(cyc)), self.h)
        return cyc.value

    def kernel_launches(self):
        return _lib.spp_kernel_launches(self.h)

    def mg_levels(self):
        return _lib.spp_mg_levels(self.h)

    def mg_level_n(self, l):
        return _lib.spp_mg_level_n(self.h, l)

    def profile_enable(self, mask=1):
        _check(_lib.spp_profile_enable(self.h, mask), self.h)

    def profile_reset(self):
        _check(_lib.spp_profile_reset(self.h), self.h)

    def dist_info(self):
        nr, dl = ctypes.c_int32(), ctypes.c_int32()
        nx, ne, by = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_double()
        _check(_lib.spp_dist_info(self.h, ctypes.byref(nr), ctypes.byref(dl), ctypes.byref(nx), ctypes.byref(by),
                                  ctypes.byref(ne)), self.h)
        return dict(nranks=nr.value, strip_levels=dl.value, xfers=nx.value, bytes=by.value, exchanges=ne.value)

    def profile(self):
        out = {}
        for k in range(PROF_CLASSES):
            n, ms, b = ctypes.c_int64(), ctypes.c_double(), ctypes.c_double()
            _lib.spp_profile_get(self.h, k, ctypes.byref(n), ctypes.byref(ms), ctypes.byref(b))
            out[_lib.spp_profile_name(k).decode()] = dict(launches=n.value, ms=ms.value, bytes=b.value)
        return out


@dataclass
class BatchResult:
    u: object
    iters: np.ndarray
    converged: np.ndarray
    res: np.ndarray
    status: int
    stats: dict


class Batch1D:
    """One spp_batch1d: nprob independent 1D problems (spp.h "Batched 1D solves").  n, eps and
    the concatenated meshes x are host arrays; c, r (and f, u at solve) are concatenated
    interior samples, numpy (host) or torch CUDA float64 (device)."""

    def __init__(self, n, eps, x, c, r, options: spp_options | None = None, stream=None):
        self.n = np.ascontiguousarray(n, dtype=np.int32)
        self.eps = np.ascontiguousarray(eps, dtype=np.float64)
        self._x = np.ascontiguousarray(x, dtype=np.float64)
        self.total = int(np.sum(self.n - 1))
        self.opt = options if options is not None else spp_default_options(1)
        if self._x.size != int(np.sum(self.n + 1)) or self.eps.size != self.n.size:
            raise SppArgError("batch: x must hold sum(N_p + 1) coordinates and eps one value per problem")
        _check_arrays([("c", c), ("r", r)], self.total)
        pc, mem, kc = _ptr(c)
        pr, _, kr = _ptr(r)
        h = _vp()
        self._stream = _stream_handle(stream)
        _check(_lib.spp_batch1d_create(len(self.n), self.n.ctypes.data_as(_ip), self.eps.ctypes.data_as(_dp),
                                       self._x.ctypes.data_as(_dp), pc, pr, mem, ctypes.byref(self.opt),
                                       self._stream, ctypes.byref(h)))
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            _lib.spp_batch1d_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def launches(self):
        return _lib.spp_batch1d_launches(self.h)

    def setup(self, c, r):
        _check_arrays([("c", c), ("r", r)], self.total)
        pc, mem, kc = _ptr(c)
        pr, _, kr = _ptr(r)
        rc = _lib.spp_batch1d_setup(self.h, pc, pr, mem)
        if rc < 0:
            raise SppError(rc, (_lib.spp_batch1d_last_error(self.h) or b"").decode())

    def solve(self, f, u=None) -> BatchResult:
        pf, mem, kf = _ptr(f)
        if u is None:
            if mem == SPP_HOST:
                u = np.zeros(self.total)
            else:
                import torch
                u = torch.zeros_like(f)
        _check_arrays([("f", f), ("u", u)], self.total)
        pu, memu, ku = _ptr(u)
        if memu != mem:
            raise ValueError("f and u must have the same residency")
        P = len(self.n)
        it, cv, res = np.zeros(P, np.int32), np.zeros(P, np.int32), np.zeros(P)
        st = spp_stats()
        rc = _lib.spp_batch1d_solve(self.h, pf, pu, mem, it.ctypes.data_as(_ip), cv.ctypes.data_as(_ip),
                                    res.ctypes.data_as(_dp), ctypes.byref(st))
        if rc < 0:
            raise SppError(rc, (_lib.spp_batch1d_last_error(self.h) or b"").decode())
        return BatchResult(u=ku if mem == SPP_HOST else u, iters=it, converged=cv.astype(bool), res=res,
                           status=rc, stats=st.asdict())


class DistSolver(Solver):
    """One row strip of a 2D problem per process (spp_create_dist): c1, c2, r (and f, u at
    solve) hold this rank's interior rows j0 .. j1-1 only; x, y are the whole meshes; comm is an
    NCCL communicator handle (nccl_comm_create).  Collective: every rank constructs and solves
    in the same order."""

    def __init__(self, n, eps, x, y, c1, c2, r, j0, j1, comm, rank, nranks, options: spp_options | None = None,
                 stream=None):
        _nccl_env()
        self.dim, self.n, self.eps, self.j0, self.j1 = 2, n, eps, j0, j1
        self.opt = options if options is not None else spp_default_options(2)
        self._x = np.ascontiguousarray(x, dtype=np.float64)
        self._y = np.ascontiguousarray(y, dtype=np.float64)
        if self._x.size != n + 1 or self._y.size != n + 1:
            raise SppArgError(f"mesh coordinates: need {n + 1} values per axis")
        _check_arrays([("c1", c1), ("c2", c2), ("r", r)], (j1 - j0) * (n - 1))
        p1, mem, k1 = _ptr(c1)
        p2, _, k2 = _ptr(c2)
        p3, _, k3 = _ptr(r)
        prob = spp_problem(2, n, eps, self._x.ctypes.data, self._y.ctypes.data, p1, p2, p3, mem)
        h = _vp()
        self._stream = _stream_handle(stream)
        _check(_lib.spp_create_dist(ctypes.byref(prob), j0, j1, comm, rank, nranks, ctypes.byref(self.opt), self._stream,
                                    ctypes.byref(h)))
        self.h = h
        self._keep = (k1, k2, k3)

    def setup(self, c1, c2, r):
        _check_arrays([("c1", c1), ("c2", c2), ("r", r)], (self.j1 - self.j0) * (self.n - 1))
        p1, mem, k1 = _ptr(c1)
        p2, _, k2 = _ptr(c2)
        p3, _, k3 = _ptr(r)
        _check(_lib.spp_setup(self.h, p1, p2, p3, mem), self.h)

    def solve(self, f, u=None, hist_cap=256) -> SolveResult:
        cnt = (self.j1 - self.j0) * (self.n - 1)
        pf, mem, kf = _ptr(f)
        if u is None:
            if mem == SPP_HOST:
                u = np.zeros(cnt)
            else:
                import torch
                u = torch.zeros_like(f)
        _check_arrays([("f", f), ("u", u)], cnt)
        pu, memu, ku = _ptr(u)
        if memu != mem:
            raise ValueError("f and u must have the same residency")
        hist = np.zeros(hist_cap)
        st = spp_stats()
        rc = _check(_lib.spp_solve(self.h, pf, pu, mem, hist.ctypes.data_as(_dp), hist_cap, ctypes.byref(st)), self.h)
        d = st.asdict()
        return SolveResult(u=ku if mem == SPP_HOST else u, hist=hist[: d["iters"] + 1].copy(), status=rc, stats=d)

"""Build the sm_100a shared library libspp.so in-tree (nvcc, no JIT cache)."""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
SRC = PKG / "csrc"
LIB = PKG / "lib" / "libspp.so"
SOURCES = ["capi.cu", "k_core.cu", "k_lines.cu", "k_1d.cu", "k_mg.cu", "dist.cu", "k_par.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
# <nccl.h> (system include path) for the types only: the library resolves NCCL at run time
# (dlopen), so libspp.so has no link dependency on it
FLAGS = [*(["-DSPP_WAVE_PROF"] if os.environ.get("SPP_WAVE_PROF") else []),
    *(["-DSPP_LINES_PROF"] if os.environ.get("SPP_LINES_PROF") else []),
    *(["-DSPP_COARSE_PROF"] if os.environ.get("SPP_COARSE_PROF") else []),
    *(["-DSPP_STRESS"] if os.environ.get("SPP_STRESS") else []),
    *([f"-D{x}" for x in os.environ.get("SPP_EXP", "").split(",") if x]), "-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
         "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden", "--expt-relaxed-constexpr",
         "-I", str(ROOT / "include"), "-I", str(SRC)]


def _stale() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    deps = [SRC / s for s in SOURCES] + list(SRC.glob("*.cuh")) + [ROOT / "include" / "spp.h", Path(__file__)]
    return any(d.stat().st_mtime > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and not _stale():
        return LIB
    LIB.parent.mkdir(exist_ok=True)
    objs = []
    for s in SOURCES:
        o = LIB.parent / (s + ".o")
        cmd = [NVCC, *FLAGS, "-dc" if False else "-c", str(SRC / s), "-o", str(o)]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.check_call(cmd)
        objs.append(str(o))
    tmp = LIB.with_suffix(f".so.tmp{os.getpid()}")
    cmd = [NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", str(tmp), *objs,
           "-Xcompiler", "-fPIC", "-cudart", "static", "-ldl"]
    subprocess.check_call(cmd)
    os.replace(tmp, LIB)
    for o in objs:
        os.remove(o)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))

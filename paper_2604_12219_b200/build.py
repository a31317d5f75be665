"""Build libpasa.so in-tree with nvcc for sm_100a (no JIT cache, no torch
extension machinery): the built library travels to the GPU box with the repo.

    python -m paper_2604_12219_b200.build [--force]
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
# A/B builds (tools/): PASA_BUILD_DIR puts objects and the library elsewhere,
# PASA_EXTRA_FLAGS adds nvcc flags (e.g. -DPASA_D64_POLY=4); the product build sets neither
_ALT = os.environ.get("PASA_BUILD_DIR")
LIBDIR = os.path.join(_ALT, "lib") if _ALT else os.path.join(PKG, "lib")
LIB = os.path.join(LIBDIR, "libpasa.so")
OBJDIR = os.path.join(_ALT, "build") if _ALT else os.path.join(PKG, "build")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2",
                 "--expt-relaxed-constexpr", "-I" + os.path.join(ROOT, "include")]
COMMON += os.environ.get("PASA_EXTRA_FLAGS", "").split()
# per-file extra flags: the route unit must not contract fp64 mul+add into fma
EXTRA = {"route.cu": ["--fmad=false"]}
SOURCES = ["api.cpp", "tmap.cpp", "budget.cu", "route.cu", "het.cu", "kv_stats.cu", "attn_simt.cu",
           "attn_sm100.cu", "attn_sm100_q256.cu", "attn_sm100_cta2.cu", "kv_stats_sm100.cu"]
HEADERS = ["pasa_internal.h", "philox.cuh", "sm100_ptx.cuh", "fastlog.cuh", "logtab.h"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _newest_dep() -> float:
    deps = [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(ROOT, "include", "pasa.h"),
                                                       os.path.abspath(__file__)]
    return max(os.path.getmtime(d) for d in deps)


def _compile(src: str, force: bool, verbose: bool) -> str:
    os.makedirs(OBJDIR, exist_ok=True)
    obj = os.path.join(OBJDIR, src + ".o")
    path = os.path.join(CSRC, src)
    if (not force and os.path.exists(obj)
            and os.path.getmtime(obj) >= max(os.path.getmtime(path), _newest_dep())):
        return obj
    cmd = [nvcc(), *COMMON, *EXTRA.get(src, []), "-c", path, "-o", obj + ".tmp"]
    if verbose and src.endswith(".cu"):
        cmd += ["-Xptxas", "-v"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{' '.join(cmd)}\n{res.stdout}\n{res.stderr}")
    if verbose and res.stderr:
        sys.stderr.write(res.stderr)
    os.replace(obj + ".tmp", obj)
    return obj


def build(force: bool = False, verbose: bool = False) -> str:
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        objs = list(ex.map(lambda s: _compile(s, force, verbose), SOURCES))
    if (force or not os.path.exists(LIB)
            or os.path.getmtime(LIB) < max(os.path.getmtime(o) for o in objs)):
        os.makedirs(LIBDIR, exist_ok=True)
        cmd = [nvcc(), *ARCH, "-shared", "--cudart=static", "-o", LIB + ".tmp", *objs, "-ldl",
               "-lpthread", "-lrt"]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"link failed:\n{' '.join(cmd)}\n{res.stdout}\n{res.stderr}")
        os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))

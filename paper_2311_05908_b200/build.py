"""In-tree build of the sm_100a shared libraries (nvcc, no torch extension).

libfftconv.so          -- the C-ABI library declared in include/fftconv.h
libfftconv_selftest.so -- device self-test hooks for the tcgen05 primitives

Both are written next to this file so they travel with the repo snapshot to
the GPU box.  Usage:  python -m paper_2311_05908_b200.build
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
INCLUDE = os.path.join(ROOT, "include")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-shared",
          "-I", INCLUDE, "-I", CSRC, "--expt-relaxed-constexpr"]

LIB = os.path.join(HERE, "libfftconv.so")
SELFTEST = os.path.join(HERE, "libfftconv_selftest.so")

LIB_SOURCES = ["plan.cpp", "api.cu", "kernels_fwd.cu", "kernels_kf.cu", "kernels_mp.cu", "kernels_bwd.cu", "kernels_f32.cu"]


def _stale(target, sources):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    deps = list(sources) + glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h")) \
        + glob.glob(os.path.join(INCLUDE, "*.h"))
    return any(os.path.getmtime(s) > t for s in deps)


def _nvcc(out, sources, extra=()):
    """Compile every source to an object in parallel, then link the shared
    library (the sources share no device symbols)."""
    from concurrent.futures import ThreadPoolExecutor
    tmp = out + f".tmp{os.getpid()}"
    objdir = os.path.join(os.path.dirname(out), "build_obj")
    os.makedirs(objdir, exist_ok=True)
    compile_flags = [f for f in COMMON if f != "-shared"]

    def one(src):
        obj = os.path.join(objdir, os.path.basename(src) + f".{os.getpid()}.o")
        subprocess.check_call([NVCC, *ARCH, *compile_flags, *extra, "-c", "-o", obj, src])
        return obj

    with ThreadPoolExecutor(max_workers=min(len(sources), os.cpu_count() or 4)) as ex:
        objs = list(ex.map(one, sources))
    subprocess.check_call([NVCC, *ARCH, "-shared", "-Xcompiler", "-fPIC", "-o", tmp, *objs])
    for o in objs:
        os.remove(o)
    os.replace(tmp, out)


def build(force: bool = False, verbose: bool = False) -> list[str]:
    built = []
    srcs = [os.path.join(CSRC, s) for s in LIB_SOURCES if os.path.exists(os.path.join(CSRC, s))]
    extra = ["-Xptxas", "-v"] if verbose else []
    if srcs and (force or _stale(LIB, srcs)):
        _nvcc(LIB, srcs, extra)
        built.append(LIB)
    st = [os.path.join(CSRC, "selftest.cu")]
    if force or _stale(SELFTEST, st):
        _nvcc(SELFTEST, st, extra)
        built.append(SELFTEST)
    return built


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))

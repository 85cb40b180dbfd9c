"""Build libqmcj2.so in-tree with nvcc for sm_100a (no JIT cache, no torch
extension machinery: the library is plain CUDA C++ with a C ABI).

Translation units are compiled to objects in parallel (the kernel
instantiations are split by dtype / mode), then linked.

Variants with extra compile flags (the -DQJ2_CHECK debug build, A/B builds
with -DQJ2_ITERS=... etc.) get their own object directory and library name,
keyed by a hash of the flags, so a variant build never stands in for the
product library or for another variant.
"""
from __future__ import annotations

import concurrent.futures as cf
import hashlib
import os
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libqmcj2.so")
LIB_CHECK = os.path.join(PKG, "libqmcj2_check.so")
OBJDIR = os.path.join(PKG, "build_obj")
SOURCES = [os.path.join(CSRC, f) for f in
           ["qmcj2.cu", "gen.cu", "launch_accept.cu", "spo.cu", "sweep.cu"] +
           [f"launch_{d}_{m}.cu" for d in ("f32", "f64") for m in ("j2", "j1")]]
HEADERS = [os.path.join(CSRC, f) for f in ("j2_device.cuh", "j2_kernels.cuh", "launch.cuh", "accept.cuh",
                                           "spo.cuh", "sweep.cuh", "bulk.cuh")] + \
          [os.path.join(ROOT, "include", "qmcj2.h")]

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-I", os.path.join(ROOT, "include")]
CHECK_FLAGS = ["-DQJ2_CHECK"]


def nvcc() -> str:
    cand = os.environ.get("NVCC")
    if cand:
        return cand
    return "/usr/local/cuda/bin/nvcc" if os.path.exists("/usr/local/cuda/bin/nvcc") else "nvcc"


def _variant(extra):
    """(object dir, library path, flags) of a build with extra flags."""
    extra = list(extra or [])
    if not extra:
        return OBJDIR, LIB, NVCC_FLAGS
    key = hashlib.sha256(" ".join(extra).encode()).hexdigest()[:10]
    lib = LIB_CHECK if extra == CHECK_FLAGS else os.path.join(PKG, f"libqmcj2_{key}.so")
    return OBJDIR + "_" + key, lib, NVCC_FLAGS + extra


def _stamp(objdir):
    return os.path.join(objdir, "FLAGS")


def up_to_date(extra=None) -> bool:
    objdir, lib, flags = _variant(extra)
    if not os.path.exists(lib) or not os.path.exists(_stamp(objdir)):
        return False
    if open(_stamp(objdir)).read() != " ".join(flags):
        return False
    t = os.path.getmtime(lib)
    return all(os.path.getmtime(d) <= t for d in SOURCES + HEADERS)


def _compile(src: str, objdir: str, flags, verbose: bool) -> str:
    obj = os.path.join(objdir, os.path.basename(src).replace(".cu", ".o"))
    hdr_t = max(os.path.getmtime(h) for h in HEADERS)
    if os.path.exists(obj) and os.path.getmtime(obj) >= max(os.path.getmtime(src), hdr_t):
        return obj
    cmd = [nvcc(), *flags, "-c", "-o", obj + f".tmp{os.getpid()}", src]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.check_call(cmd)
    os.replace(obj + f".tmp{os.getpid()}", obj)
    return obj


def build(force: bool = False, verbose: bool = False, extra=None) -> str:
    """Build the library (extra: additional nvcc flags -> a separate variant);
    returns its path.  QJ2_EXTRA_FLAGS (environment) adds flags too."""
    extra = list(extra or []) + os.environ.get("QJ2_EXTRA_FLAGS", "").split()
    objdir, lib, flags = _variant(extra)
    if not force and up_to_date(extra):
        return lib
    os.makedirs(objdir, exist_ok=True)
    stamp = _stamp(objdir)
    if force or not os.path.exists(stamp) or open(stamp).read() != " ".join(flags):
        for f in os.listdir(objdir):
            if f.endswith(".o"):
                os.remove(os.path.join(objdir, f))
    with cf.ThreadPoolExecutor(max_workers=min(len(SOURCES), os.cpu_count() or 1)) as ex:
        objs = list(ex.map(lambda s: _compile(s, objdir, flags, verbose), SOURCES))
    tmp = lib + f".tmp{os.getpid()}"
    cmd = [nvcc(), *ARCH, "-shared", "-o", tmp, *objs]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.check_call(cmd)
    os.replace(tmp, lib)
    with open(stamp, "w") as f:
        f.write(" ".join(flags))
    return lib


def build_check(force: bool = False, verbose: bool = False) -> str:
    """The -DQJ2_CHECK debug build (device-side index checks), libqmcj2_check.so."""
    return build(force=force, verbose=verbose, extra=CHECK_FLAGS)


if __name__ == "__main__":
    print(build(force=True, verbose=True))
    print(build_check(force=True, verbose=True))

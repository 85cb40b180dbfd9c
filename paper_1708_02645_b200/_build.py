"""Build libqmcj2.so in-tree with nvcc for sm_100a (no JIT cache, no torch
extension machinery: the library is plain CUDA C++ with a C ABI).

Translation units are compiled to objects in parallel (the kernel
instantiations are split by dtype / trial-batch size), then linked."""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libqmcj2.so")
OBJDIR = os.path.join(PKG, "build_obj")
SOURCES = [os.path.join(CSRC, f) for f in
           ["qmcj2.cu", "gen.cu", "launch_accept.cu", "spo.cu", "sweep.cu"] + [f"launch_{d}_{b}_{m}.cu" for d in ("f32", "f64") for b in ("pb1",)
                                     for m in ("j2", "j1")]]
HEADERS = [os.path.join(CSRC, f) for f in ("j2_device.cuh", "j2_kernels.cuh", "j2_tma.cuh", "launch.cuh", "accept.cuh", "spo.cuh", "sweep.cuh", "bulk.cuh")] + \
          [os.path.join(ROOT, "include", "qmcj2.h")]

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-I", os.path.join(ROOT, "include")]
# A/B builds only (e.g. QJ2_EXTRA_FLAGS="-DQJ2_SWEEP_MINB128=7" with build(force=True))
NVCC_FLAGS += os.environ.get("QJ2_EXTRA_FLAGS", "").split()


def nvcc() -> str:
    cand = os.environ.get("NVCC")
    if cand:
        return cand
    return "/usr/local/cuda/bin/nvcc" if os.path.exists("/usr/local/cuda/bin/nvcc") else "nvcc"


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(d) <= t for d in SOURCES + HEADERS)


def _obj(src: str) -> str:
    return os.path.join(OBJDIR, os.path.basename(src).replace(".cu", ".o"))


def _compile(src: str, verbose: bool) -> str:
    obj = _obj(src)
    hdr_t = max(os.path.getmtime(h) for h in HEADERS)
    if os.path.exists(obj) and os.path.getmtime(obj) >= max(os.path.getmtime(src), hdr_t):
        return obj
    cmd = [nvcc(), *NVCC_FLAGS, "-c", "-o", obj + f".tmp{os.getpid()}", src]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.check_call(cmd)
    os.replace(obj + f".tmp{os.getpid()}", obj)
    return obj


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and up_to_date():
        return LIB
    os.makedirs(OBJDIR, exist_ok=True)
    if force:
        for s in SOURCES:
            if os.path.exists(_obj(s)):
                os.remove(_obj(s))
    with cf.ThreadPoolExecutor(max_workers=min(len(SOURCES), os.cpu_count() or 1)) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose), SOURCES))
    tmp = LIB + f".tmp{os.getpid()}"
    cmd = [nvcc(), *ARCH, "-shared", "-o", tmp, *objs]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.check_call(cmd)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force=True, verbose=True))

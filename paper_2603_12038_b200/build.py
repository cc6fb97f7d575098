"""In-tree build of the sm_100a extension.

  libsfi_b200.so       C ABI (include/sfi_b200.h) + C++ host API
                       (include/sfi_b200.hpp) + all CUDA kernels, cudart static
  _sfi_b200*.so        pybind11 module over the C++ host API (rpath $ORIGIN)

Every CUDA translation unit is compiled with
``-gencode arch=compute_100a,code=sm_100a -lineinfo``; selector.cu also gets
``-fmad=false`` (no FMA contraction, matching the reference's fp64 rounding).
Incremental: a target is rebuilt when any of its inputs is newer.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys
import sysconfig

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INC = os.path.join(ROOT, "include")
OBJ = os.path.join(ROOT, "build", "obj")
LIB = os.path.join(PKG, "libsfi_b200.so")
EXT = os.path.join(PKG, "_sfi_b200" + sysconfig.get_config_var("EXT_SUFFIX"))
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-fvisibility=hidden",
                 "-I" + INC, "-I" + CSRC]
CU = ["decode.cu", "fast_decode.cu", "capture.cu", "cache_ops.cu", "selector.cu", "capi.cu"]
CPP = ["host.cpp", "engine.cpp"]
HEADERS = [os.path.join(INC, h) for h in ("sfi_b200.h", "sfi_b200.hpp")] + [
    os.path.join(CSRC, h) for h in ("common.cuh", "kernels.h")]


def _newer(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _run(cmd: list[str]) -> None:
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("build failed: " + " ".join(cmd[:6]) + " ...")


def _compile(src: str) -> str:
    path = os.path.join(CSRC, src)
    obj = os.path.join(OBJ, src + ".o")
    if _newer(obj, [path] + HEADERS):
        extra = ["-fmad=false"] if src == "selector.cu" else []
        if src == "engine.cpp":  # the toy model's fp64 host math: no contraction, as in the reference build
            extra = ["-Xcompiler", "-ffp-contract=off"]
        _run([NVCC] + COMMON + extra + ["-c", path, "-o", obj])
    return obj


def build(verbose: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    with cf.ThreadPoolExecutor(max_workers=len(CU) + len(CPP)) as ex:
        objs = list(ex.map(_compile, CU + CPP))
    if _newer(LIB, objs):
        _run([NVCC] + ARCH + ["-shared", "-cudart", "static", "-o", LIB] + objs +
             ["-Xlinker", "--exclude-libs,ALL"])
    bsrc = os.path.join(CSRC, "bindings.cpp")
    if _newer(EXT, [bsrc, LIB] + HEADERS):
        import pybind11
        _run(["g++", "-O2", "-std=c++17", "-shared", "-fPIC", "-fvisibility=hidden",
              "-I" + pybind11.get_include(), "-I" + sysconfig.get_paths()["include"], "-I" + INC,
              bsrc, "-o", EXT, "-L" + PKG, "-lsfi_b200", "-Wl,-rpath,$ORIGIN"])
    if verbose:
        print("built", LIB, EXT)
    return EXT


if __name__ == "__main__":
    build(verbose=True)

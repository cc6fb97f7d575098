"""In-tree build of the sm_100a extension.

  libsfi_b200.so       C ABI (include/sfi_b200.h) + C++ host API
                       (include/sfi/*.hpp, namespace sfi) + all CUDA kernels,
                       cudart static
  _sfi_b200*.so        pybind11 module over the C++ host API (rpath $ORIGIN)
  harness/libsfi_toy.so, harness/_sfi_toy*.so
                       END-TO-END TEST HARNESS (not product): the toy decoder
                       + request loop (harness/engine.cpp) over libsfi_b200.so

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
HARNESS = os.path.join(ROOT, "harness")
TOY_LIB = os.path.join(HARNESS, "libsfi_toy.so")
TOY_EXT = os.path.join(HARNESS, "_sfi_toy" + sysconfig.get_config_var("EXT_SUFFIX"))
CU = ["decode.cu", "fast_decode.cu", "capture.cu", "cache_ops.cu", "selector.cu", "capi.cu"]
CPP = ["host.cpp", "executor.cpp"]
HEADERS = [os.path.join(INC, h) for h in ("sfi_b200.h", "sfi_b200.hpp")] + [
    os.path.join(INC, "sfi", h) for h in ("attention.hpp", "config.hpp", "decode.hpp", "distribution.hpp", "error.hpp",
                                          "scheduler.hpp", "selector.hpp")] + [
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
        cmd = [NVCC] + COMMON + extra + ["-c", path, "-o", obj]
        if src.endswith(".cpp"):  # the host API is C++20 (std::span, as the reference's headers)
            cmd = [NVCC] + ARCH + ["-O3", "-std=c++20", "-Xcompiler", "-fPIC,-fvisibility=hidden",
                                   "-I" + INC, "-I" + CSRC, "-c", path, "-o", obj]
        _run(cmd)
    return obj


def build(verbose: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    with cf.ThreadPoolExecutor(max_workers=len(CU) + len(CPP)) as ex:
        objs = list(ex.map(_compile, CU + CPP))
    if _newer(LIB, objs):
        _run([NVCC] + ARCH + ["-shared", "-cudart", "static", "-o", LIB] + objs +
             ["-Xlinker", "--exclude-libs,ALL"])
    import pybind11
    py_inc = ["-I" + pybind11.get_include(), "-I" + sysconfig.get_paths()["include"], "-I" + INC]
    bsrc = os.path.join(CSRC, "bindings.cpp")
    if _newer(EXT, [bsrc, LIB] + HEADERS):
        _run(["g++", "-O2", "-std=c++20", "-shared", "-fPIC", "-fvisibility=hidden"] + py_inc +
             [bsrc, "-o", EXT, "-L" + PKG, "-lsfi_b200", "-Wl,-rpath,$ORIGIN"])
    # test harness: the toy decoder + request loop over the product library
    esrc, tsrc, thdr = (os.path.join(HARNESS, f) for f in ("engine.cpp", "toy_bindings.cpp", "sfi_toy.hpp"))
    cuda_inc = "-I" + os.path.join(os.path.dirname(os.path.dirname(NVCC)), "include")
    if _newer(TOY_LIB, [esrc, thdr, LIB] + HEADERS):
        # the toy model's fp64 host math: no contraction, as in the reference build
        _run(["g++", "-O2", "-std=c++20", "-shared", "-fPIC", "-ffp-contract=off", "-I" + INC, "-I" + HARNESS,
              cuda_inc, esrc, "-o", TOY_LIB, "-L" + PKG, "-lsfi_b200", "-Wl,-rpath,$ORIGIN/../paper_2603_12038_b200",
              "-L" + os.path.join(os.path.dirname(os.path.dirname(NVCC)), "lib64"), "-lcudart"])
    if _newer(TOY_EXT, [tsrc, thdr, TOY_LIB] + HEADERS):
        _run(["g++", "-O2", "-std=c++20", "-shared", "-fPIC", "-fvisibility=hidden"] + py_inc +
             ["-I" + HARNESS, tsrc, "-o", TOY_EXT, "-L" + HARNESS, "-lsfi_toy", "-L" + PKG, "-lsfi_b200",
              "-Wl,-rpath,$ORIGIN", "-Wl,-rpath,$ORIGIN/../paper_2603_12038_b200"])
    if verbose:
        print("built", LIB, EXT, TOY_LIB, TOY_EXT)
    return EXT


if __name__ == "__main__":
    build(verbose=True)

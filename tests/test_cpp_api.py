"""The reference's C++ call sites compile and run against the reference's own
header paths (include/sfi/*.hpp, namespace sfi) and libsfi_b200.so
(tests/cpp/test_api.cpp): host cases on CPU; device cases (KvStore's reference
surface — key_at views, compact() by const reference, general sinks, a recent
range that is not the tail, the access trace — reorganize, the Selector stage
functions, run_selector with a SelectorTrace, select_top_k KATs) on the B200.
tests/cpp/test_toy.cpp runs the run_request / run_dense request loop (C7, C8)
against the test harness library (harness/libsfi_toy.so)."""
from __future__ import annotations

import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "test_api.cpp")
LIBDIR = os.path.join(ROOT, "paper_2603_12038_b200")
BIN = os.path.join(ROOT, "build", "test_api")


HARNESS = os.path.join(ROOT, "harness")
TOY_SRC = os.path.join(ROOT, "tests", "cpp", "test_toy.cpp")
TOY_BIN = os.path.join(ROOT, "build", "test_toy")


def _compile(src, out, extra):
    os.makedirs(os.path.dirname(out), exist_ok=True)
    libs = [os.path.join(LIBDIR, "libsfi_b200.so")] + [os.path.join(HARNESS, "libsfi_toy.so")] * ("-lsfi_toy" in extra)
    if not os.path.exists(out) or os.path.getmtime(out) < max(os.path.getmtime(x) for x in [src] + libs):
        r = subprocess.run(["g++", "-std=c++20", "-O1", "-I" + os.path.join(ROOT, "include"), src, "-o", out,
                            "-L" + LIBDIR, "-lsfi_b200", "-Wl,-rpath," + LIBDIR] + extra,
                           capture_output=True, text=True)
        assert r.returncode == 0, r.stderr
    return out


@pytest.fixture(scope="module")
def binary():
    return _compile(SRC, BIN, [])


def test_cpp_host_api(binary):
    r = subprocess.run([binary], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.gpu
def test_cpp_device_api(binary):
    r = subprocess.run([binary, "gpu"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.gpu
def test_cpp_toy_request_loop():
    binary = _compile(TOY_SRC, TOY_BIN, ["-I" + HARNESS, "-L" + HARNESS, "-lsfi_toy", "-Wl,-rpath," + HARNESS])
    r = subprocess.run([binary], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr

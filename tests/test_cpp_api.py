"""The reference's C++ call sites compile and run against include/sfi_b200.hpp
and libsfi_b200.so (tests/cpp/test_api.cpp): host cases on CPU, device cases
(KvStore::reorganize, run_selector, select_top_k KATs, the run_request / run_dense
request loop with C7 and C8) on the B200."""
from __future__ import annotations

import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "test_api.cpp")
LIBDIR = os.path.join(ROOT, "paper_2603_12038_b200")
BIN = os.path.join(ROOT, "build", "test_api")


@pytest.fixture(scope="module")
def binary():
    os.makedirs(os.path.dirname(BIN), exist_ok=True)
    if not os.path.exists(BIN) or os.path.getmtime(BIN) < max(os.path.getmtime(SRC),
                                                                os.path.getmtime(os.path.join(LIBDIR, "libsfi_b200.so"))):
        r = subprocess.run(["g++", "-std=c++17", "-O1", "-I" + os.path.join(ROOT, "include"), SRC, "-o", BIN,
                            "-L" + LIBDIR, "-lsfi_b200", "-Wl,-rpath," + LIBDIR],
                           capture_output=True, text=True)
        assert r.returncode == 0, r.stderr
    return BIN


def test_cpp_host_api(binary):
    r = subprocess.run([binary], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.gpu
def test_cpp_device_api(binary):
    r = subprocess.run([binary, "gpu"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr

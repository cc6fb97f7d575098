"""CPU: the C-ABI library loads and exports every symbol include/sfi_b200.h
declares; the host-only entry points behave (no device needed)."""
from __future__ import annotations

import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "sfi_b200.h")
LIB = os.path.join(ROOT, "paper_2603_12038_b200", "libsfi_b200.so")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"SFI_API\s+[\w\s\*]+?\b(sfi_\w+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(LIB):
        pytest.fail("libsfi_b200.so not built; run __graft_entry__.build()")
    return C.CDLL(LIB)


def test_every_declared_symbol_is_exported(lib):
    syms = declared_symbols()
    assert len(syms) >= 20
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing


def test_binary_targets_sm100a():
    import subprocess

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", LIB], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out, out[:400]


class Shape(C.Structure):
    _fields_ = [(n, C.c_int32) for n in ("n_layers", "batch", "n_kv_heads", "n_q_heads", "head_dim",
                                          "max_positions", "n_sink", "k_budget", "n_recent")]


class Sizes(C.Structure):
    _fields_ = [(n, C.c_size_t) for n in ("kv_cache", "key_norms", "compact", "sel", "n_sel",
                                           "per_batch", "workspace", "pooled_logits")]


def _shape(**kw):
    d = dict(n_layers=36, batch=8, n_kv_heads=8, n_q_heads=32, head_dim=128, max_positions=33000,
             n_sink=4, k_budget=2048, n_recent=256)
    d.update(kw)
    return Shape(**d)


def test_shape_validation_and_sizes(lib):
    lib.sfi_last_error.restype = C.c_char_p
    s = _shape()
    assert lib.sfi_shape_validate(C.byref(s)) == 0
    z = Sizes()
    assert lib.sfi_buffer_sizes(C.byref(s), C.byref(z)) == 0
    slices = 36 * 8 * 8
    assert z.kv_cache == slices * 33000 * 128 * 2
    assert z.compact == slices * (256 + 4 + 2048) * 128 * 2
    assert z.key_norms == slices * 33000 * 8
    assert lib.sfi_shape_validate(C.byref(_shape(n_q_heads=33))) == 1  # config
    assert b"multiple" in lib.sfi_last_error()
    assert lib.sfi_shape_validate(C.byref(_shape(head_dim=96))) == 101  # unsupported
    assert lib.sfi_shape_validate(C.byref(_shape(n_q_heads=8 * 32))) == 101  # G = 32


def test_recent_window_matches_scheduler_rule(lib):
    rs, rl = C.c_int32(), C.c_int32()
    for prefix in (1, 2, 4, 6, 12, 40, 300):
        lib.sfi_recent_window(prefix, min(4, prefix), 8, C.byref(rs), C.byref(rl))
        want = max(0, min(8, prefix - min(4, prefix)))
        assert rl.value == want and rs.value == prefix - want + 1


def test_device_calls_fail_cleanly_without_buffers(lib):
    s = _shape()
    assert lib.sfi_dense_decode(C.byref(s), None, 0, None, None, None, 0, None) == 102
    assert lib.sfi_step_advance(None, None, None) == 102

"""B200-native Slow-Fast Inference (SFI, arXiv 2603.12038) decode-attention hot path.

The reference's operator API (``sfi`` python module, proj/python/sfi/__init__.py)
re-implemented on sm_100a: every hot-path call below launches the CUDA kernels
in ``libsfi_b200.so`` through the C ABI (include/sfi_b200.h). There is no CPU
fallback: importing this package fails loudly when the extension is missing.

Reference-named operators (hot path):
    run_selector, select_top_k, make_cache_stats, KvStore,
    attention_kernel_dense, attention_kernel_sparse, dense_capture
Host-side scheduler bookkeeping (integer logic, scheduler.cpp):
    init_decode_state, compute_allowed, next_step_type,
    fast_step_update, slow_step_update, flop_model
Request loop around the device path (scheduler.cpp:213-365), with the
reference's toy decoder as the activation source:
    ToyModel, run_request, run_dense, argmax_token
Batched device API (production / bench): SfiCache (torch-allocated buffers).
"""
from __future__ import annotations

import os as _os

_HERE = _os.path.dirname(_os.path.abspath(__file__))

try:
    from . import _sfi_b200 as _C  # noqa: F401
except ImportError as _e:  # pragma: no cover - exercised only on broken installs
    raise ImportError(
        "paper_2603_12038_b200: the sm_100a extension is not built "
        f"({_e}); run `python -c 'import __graft_entry__ as g; g.build()'` "
        "or `python paper_2603_12038_b200/build.py`") from _e

from ._sfi_b200 import (  # noqa: F401,E402
    CacheLimits,
    CacheStats,
    CompactSegment,
    Config,
    DecodeState,
    DenseCapture,
    KernelStats,
    KvStore,
    LogitWindow,
    ModelSpec,
    PoolMode,
    RequestResult,
    RunOptions,
    SelectorConfig,
    SelectorParams,
    SelectorStages,
    SfiError,
    SparseState,
    StepCause,
    StepRecord,
    SupportSet,
    ToyModel,
    TriggerConfig,
    argmax_token,
    attention_kernel_dense,
    attention_kernel_sparse,
    compute_allowed,
    default_config,
    dense_capture,
    fast_step_update,
    flop_model,
    init_decode_state,
    make_cache_stats,
    next_step_type,
    run_dense,
    run_request,
    run_selector,
    run_selector_stages,
    select_top_k,
    slow_step_update,
)

LIBRARY_PATH = _os.path.join(_HERE, "libsfi_b200.so")


def __getattr__(name):
    if name in ("SfiCache", "SlowStepPipeline"):
        from . import device

        return getattr(device, name)
    raise AttributeError(name)


__all__ = [
    "CacheLimits", "CacheStats", "CompactSegment", "Config", "DecodeState", "DenseCapture",
    "KernelStats", "KvStore", "LogitWindow", "ModelSpec", "PoolMode", "SelectorConfig",
    "SelectorParams", "SelectorStages", "SfiError", "SparseState", "SupportSet", "TriggerConfig",
    "attention_kernel_dense", "attention_kernel_sparse", "compute_allowed", "default_config",
    "dense_capture", "fast_step_update", "flop_model", "init_decode_state", "make_cache_stats",
    "next_step_type", "run_selector", "run_selector_stages", "select_top_k", "slow_step_update",
    "SfiCache", "SlowStepPipeline", "LIBRARY_PATH",
    "ToyModel", "StepCause", "StepRecord", "RunOptions", "RequestResult", "run_request", "run_dense",
    "argmax_token",
]

"""B200-native Slow-Fast Inference (SFI, arXiv 2603.12038) decode-attention hot path.

The reference's operator API (``sfi`` python module, proj/python/sfi/__init__.py)
re-implemented on sm_100a: every hot-path call below launches the CUDA kernels
in ``libsfi_b200.so`` through the C ABI (include/sfi_b200.h). There is no CPU
fallback: importing this package fails loudly when the extension is missing.

Reference names (``sfi._sfi``):
    Selector: run_selector, evidence_from_window, prior_from_stats, fuse,
        refine_soft_nms, refine_cross_head, select_top_k, make_cache_stats,
        normalize, validate_distribution, ScoreDistribution, FusedScore
        (every stage on the device)
    KV / attention: KvStore, attention_kernel_dense, attention_kernel_sparse
    Config: SelectorConfig, TriggerConfig, CacheLimits, Config, default_config,
        load_config_file, save_config_file
    Scheduler bookkeeping (host integer logic, scheduler.cpp): init_decode_state,
        compute_allowed, next_step_type, fast_step_update, slow_step_update,
        flop_model, StepRecord
B200 additions: dense_capture (the slow-step capture as an operator),
SfiCache (batched device API over torch-allocated buffers, the production /
bench path), SlowStepPipeline, sharded.HeadShardedSfi / SeqShardedSfi.
The reference's toy decoder and request loop (ToyModel, run_request,
run_dense) are end-to-end TEST HARNESS code, in the separate ``harness``
package (harness/libsfi_toy.so), not in this library.
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
    FusedScore,
    KernelStats,
    KvStore,
    LogitWindow,
    ModelSpec,
    PoolMode,
    RefinedScores,
    ScoreDistribution,
    SelectorConfig,
    SelectorParams,
    SelectorTrace,
    SfiError,
    SparseState,
    StepCause,
    StepRecord,
    SupportSet,
    TriggerConfig,
    attention_kernel_dense,
    attention_kernel_sparse,
    compute_allowed,
    default_config,
    dense_capture,
    dot,
    evidence_from_window,
    fast_step_update,
    flop_model,
    fuse,
    init_decode_state,
    load_config_file,
    make_cache_stats,
    next_step_type,
    normalize,
    prior_from_stats,
    refine_cross_head,
    refine_soft_nms,
    run_selector,
    same_support,
    save_config_file,
    select_top_k,
    slow_step_update,
    squared_norm,
    step_record_to_json,
    validate_distribution,
)

LIBRARY_PATH = _os.path.join(_HERE, "libsfi_b200.so")


def __getattr__(name):
    if name in ("SfiCache", "SlowStepPipeline"):
        from . import device

        return getattr(device, name)
    raise AttributeError(name)


__all__ = [
    "CacheLimits", "CacheStats", "CompactSegment", "Config", "DecodeState", "DenseCapture", "FusedScore",
    "KernelStats", "KvStore", "LogitWindow", "ModelSpec", "PoolMode", "RefinedScores", "ScoreDistribution",
    "SelectorConfig", "SelectorParams", "SelectorTrace", "SfiError", "SparseState", "StepCause", "StepRecord",
    "SupportSet", "TriggerConfig", "attention_kernel_dense", "attention_kernel_sparse", "compute_allowed",
    "default_config", "dense_capture", "dot", "evidence_from_window", "fast_step_update", "flop_model", "fuse",
    "init_decode_state", "load_config_file", "make_cache_stats", "next_step_type", "normalize",
    "prior_from_stats", "refine_cross_head", "refine_soft_nms", "run_selector", "same_support",
    "save_config_file", "select_top_k", "slow_step_update", "squared_norm", "step_record_to_json",
    "validate_distribution", "SfiCache", "SlowStepPipeline", "LIBRARY_PATH",
]

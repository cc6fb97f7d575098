"""Shared test helpers: bf16 rounding, seeded inputs, and oracle stores built
from device cache contents (the oracle is the checker; tests only)."""
from __future__ import annotations

import numpy as np

from oracle import oracle as O


def bf16_round(x) -> np.ndarray:
    """Round-to-nearest-even fp32 -> bf16, returned as fp32 (exactly representable)."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    u = x.view(np.uint32).astype(np.uint64)
    u = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return u.astype(np.uint32).view(np.float32).reshape(x.shape)


def oracle(kind: str = "best") -> O.Oracle:
    return O.load(kind)


def store_from_rows(orc: O.Oracle, k_rows, v_rows, Hq: int, extra: int = 8) -> O.Store:
    """One-layer oracle KvStore from per-head rows k_rows[h][pos-1][d] (fp32),
    with room for `extra` more appended tokens."""
    k_rows = np.asarray(k_rows, np.float32)
    v_rows = np.asarray(v_rows, np.float32)
    H, L, d = k_rows.shape
    st = orc.store(1, H, Hq, d, max(L, 1) + extra)
    # [H][L][d] -> [L][H*d]
    st.append_many(np.transpose(k_rows, (1, 0, 2)).reshape(L, H * d),
                   np.transpose(v_rows, (1, 0, 2)).reshape(L, H * d))
    return st


def rel_err(got, want) -> float:
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    scale = max(np.abs(want).max(), 1e-30)
    return float(np.abs(got - want).max() / scale)

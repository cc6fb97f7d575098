"""K1 on tcgen05 vs the mma.sync kernel and the oracle: outputs, pooled logits
and timing per G (probe; the parity tests are tests/test_decode_tc.py)."""
import sys
import os
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_12038_b200 import SfiCache  # noqa: E402


def case(B, H, Hq, lens, pool, seed=1, timing=False):
    c = SfiCache(1, B, H, Hq, 128, max(lens) + 8, 4, 64, 32)
    c.fill_synthetic(seed=seed, length=max(lens))
    c.set_lengths(lens, [4] * B)
    q = torch.randn(B, Hq, 128, generator=torch.Generator().manual_seed(seed)).cuda()
    res = {}
    for k in ("mma", "tc"):
        out = torch.zeros_like(q)
        lg = torch.full_like(c.pooled_logits, float("nan"))
        c.dense_decode_ex(0, q, out, lg, pool, kernel=k)
        torch.cuda.synchronize()
        c.check_errors()
        res[k] = (out, lg)
        if timing:
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            for _ in range(3):
                c.dense_decode_ex(0, q, out, lg, pool, kernel=k)
            a.record()
            for _ in range(10):
                c.dense_decode_ex(0, q, out, lg, pool, kernel=k)
            b.record()
            torch.cuda.synchronize()
            ms = a.elapsed_time(b) / 10
            nbytes = sum(lens) * H * 512
            res[k + "_ms"] = ms
            res[k + "_gbs"] = nbytes / ms / 1e6
    o1, l1 = res["mma"]
    o2, l2 = res["tc"]
    e_o = float((o1 - o2).abs().max() / o1.abs().max())
    m = ~torch.isnan(l1)
    e_l = float((l1[m] - l2[m]).abs().max() / l1[m].abs().max()) if m.any() else 0.0
    nan_mismatch = int((torch.isnan(l1) != torch.isnan(l2)).sum())
    print(f"B={B} H={H} Hq={Hq} lens={lens} pool={pool}: out rel {e_o:.2e} logits rel {e_l:.2e} nan-mismatch {nan_mismatch}",
          {k: round(v, 1) for k, v in res.items() if k.endswith("_ms") or k.endswith("_gbs")}, flush=True)
    return e_o, e_l


if __name__ == "__main__":
    torch.cuda.set_device(0)
    for G in (4, 8, 16):
        H = 8 if G < 16 else 4
        case(1, H, H * G, [200], 0)
        case(2, H, H * G, [1000, 777], 1)
        case(3, H, H * G, [5000, 129, 4096], 0)
    case(8, 8, 32, [32768] * 8, 0, timing=True)
    case(4, 8, 64, [131072] * 4, 0, timing=True)
    case(1, 4, 64, [262144], 0, timing=True)
    # ragged: one slice over (almost) every CTA -> the one-warp merge fallback
    case(2, 4, 64, [262144, 300], 0)
    case(2, 8, 32, [200000, 64], 1)

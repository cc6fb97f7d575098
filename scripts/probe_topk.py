"""Selector timing per config with the top-k variant chosen by the environment
(SFI_TOPK_BT=1: the rows x segments histogram top-k at every length; =0: the
single-CTA / cluster top-k), one layer, logits from the dense decode of peaked
inputs. Prints ms per Selector call (queued back to back, CUDA events) and a
checksum of the selected indices so two runs can be compared.

    SFI_TOPK_BT=1 python scripts/probe_topk.py c2 c3 c4
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2603_12038_b200 as sfi  # noqa: E402


def run(cfg):
    name, L, Hq, H, B, ctx, ns, K, R = bench.CONFIGS[cfg]
    c = sfi.SfiCache(1, B, H, Hq, 128, ctx + 64, ns, K, R)
    c.fill_synthetic(seed=7, length=ctx)
    c.set_lengths([ctx] * B, [ns] * B)
    q = torch.randn(B, Hq, 128, generator=torch.Generator().manual_seed(3)).cuda()
    c.plant_peaked(0, q, n_planted=32, scale=3.0, seed=11)
    out = torch.zeros_like(q)
    logits = torch.zeros_like(c.pooled_logits)
    c.dense_decode(0, q, out, logits, 0)
    prm = sfi.SelectorParams()
    c.selector(0, logits, prm)
    torch.cuda.synchronize()
    c.check_errors()
    sel = c.sel[0].cpu().numpy().tobytes() + c.n_sel[0].cpu().numpy().tobytes()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 20
    a.record()
    for _ in range(reps):
        c.selector(0, logits, prm)
    b.record()
    torch.cuda.synchronize()
    c.check_errors()
    return {"config": cfg, "bt": os.environ.get("SFI_TOPK_BT"), "selector_us": a.elapsed_time(b) / reps * 1e3,
            "sel_sha": hashlib.sha1(sel).hexdigest()[:16]}


if __name__ == "__main__":
    for cfg in sys.argv[1:] or ["c2", "c3", "c4"]:
        print(json.dumps(run(cfg)), flush=True)
        torch.cuda.empty_cache()

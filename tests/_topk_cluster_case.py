"""Child process of tests/test_baseline_parity.py::test_forced_cluster_topk.

SFI_TOPK_CLUSTER (read once per process by the Selector's top-k launcher) forces
the cluster top-k: =1 the 8-CTA variant, =4 the 4-CTA one, for every row length;
SFI_TOPK_BT=1 forces the rows x segments histogram top-k (sel_bt_*) instead.
Runs the device Selector in cache mode at |J| ~ 5K (keys in shared memory) and
~100K (4-CTA: 25K keys per CTA > the 22K shared-memory cap, so global keys) and
compares the indices with the reference run_selector. Prints "ok".
"""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))


def main() -> None:
    import torch

    from helpers import oracle
    from oracle import oracle as O
    from paper_2603_12038_b200 import SelectorParams, SfiCache

    assert os.environ.get("SFI_TOPK_CLUSTER") in ("1", "4") or os.environ.get("SFI_TOPK_BT") == "1"
    for B, H, Hq, lens, K in [(2, 4, 16, [5300, 4100], 700), (1, 8, 32, [100_400], 2048)]:
        c = SfiCache(1, B, H, Hq, 128, max(lens) + 8, 4, K, 256)
        c.fill_synthetic(seed=max(lens), length=max(lens))
        c.set_lengths(lens, [4] * B)
        q = torch.randn(B, Hq, 128, generator=torch.Generator().manual_seed(B)).cuda()
        out = torch.zeros_like(q)
        lg = torch.zeros_like(c.pooled_logits)
        c.dense_decode(0, q, out, lg, 0)
        c.selector(0, lg, SelectorParams())
        torch.cuda.synchronize()
        c.check_errors()
        for b in range(B):
            L, rl = int(c.prefix_len[b]), int(c.recent_len[b])
            j0, j1 = 5, L - rl
            vals = lg[b, :, :j1 - j0 + 1].double().cpu().numpy()
            norms = c.key_norms[0, b, :, j0 - 1:j1].cpu().numpy()
            want, _ = oracle().run_selector(vals, np.arange(j0, j1 + 1), norms, O.make_cfg(k_budget=K))
            for h in range(H):
                got = c.sel[0, b, h, :int(c.n_sel[0, b, h])].cpu().numpy()
                assert np.array_equal(got, want[h]), (lens, b, h)
    print("ok")


if __name__ == "__main__":
    main()

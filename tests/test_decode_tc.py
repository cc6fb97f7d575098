"""K1 on the 5th-generation tensor cores (decode_tc_kernel: tcgen05.mma with
S^T / O^T accumulators in TMEM) against the CPU oracle and the mma.sync kernel:
dense attention outputs and pooled logits (mean / max) within 2e-3 of the
port's run_step capture (pinned to the reference, tests/test_oracle.py), for
G = 4, 8, 16, ragged batches, slices split over many CTAs (merge path),
slices far larger than one CTA's range (the one-warp merge fallback), and
the partial (O, LSE) mode of sequence shards."""
from __future__ import annotations

import numpy as np
import pytest

from helpers import oracle, rel_err, store_from_rows

pytestmark = pytest.mark.gpu
TOL = 2e-3


@pytest.mark.parametrize("H,Hq,lens,pool", [
    (8, 32, [700, 650], 0),             # G = 4
    (8, 64, [1500, 129, 4000], 1),      # G = 8, ragged incl. one tile + 1
    (4, 64, [900, 300], 0),             # G = 16 (Qwen3-235B group)
    (2, 32, [9000], 1),                 # G = 16, one slice over many CTAs
    (4, 64, [40000, 100], 0),           # a slice over ~all CTAs: merge fallback
])
def test_dense_tc_matches_oracle(H, Hq, lens, pool):
    import torch

    from paper_2603_12038_b200 import SfiCache

    B = len(lens)
    c = SfiCache(1, B, H, Hq, 128, max(lens) + 8, 4, 64, 32)
    c.fill_synthetic(seed=H * Hq + len(lens), length=max(lens))
    c.set_lengths(lens, [4] * B)
    q = torch.randn(B, Hq, 128, generator=torch.Generator().manual_seed(Hq + pool))
    out = torch.zeros(B, Hq, 128, device="cuda")
    lg = torch.zeros_like(c.pooled_logits)
    c.dense_decode_ex(0, q.cuda(), out, lg, pool, kernel="tc")
    out_m = torch.zeros_like(out)
    lg_m = torch.zeros_like(lg)
    c.dense_decode_ex(0, q.cuda(), out_m, lg_m, pool, kernel="mma")
    torch.cuda.synchronize()
    c.check_errors()
    port = oracle("port")
    for b in range(B):
        L, rl = int(c.prefix_len[b]), int(c.recent_len[b])
        j0, j1 = 5, L - rl
        k = c.k_cache[0, b, :, :L].float().cpu().numpy()
        v = c.v_cache[0, b, :, :L].float().cpu().numpy()
        want_o, want_lg = store_from_rows(port, k, v, Hq).dense_capture(
            0, q[b].double().numpy(), np.arange(j0, j1 + 1), pool)
        assert rel_err(out[b].cpu().numpy().reshape(-1), want_o) < TOL, b
        if j1 >= j0:
            assert rel_err(lg[b, :, :j1 - j0 + 1].cpu().numpy(), want_lg) < TOL, b
    assert rel_err(out.cpu().numpy(), out_m.cpu().numpy()) < 1e-4


def test_dense_tc_partial_mode_lse():
    """Sequence-shard partial mode: (O, LSE) of the tcgen05 kernel == the mma.sync kernel's."""
    import torch

    from paper_2603_12038_b200 import SfiCache

    B, H, Hq, lens = 2, 4, 64, [3000, 1700]
    c = SfiCache(1, B, H, Hq, 128, max(lens) + 8, 4, 64, 32)
    c.fill_synthetic(seed=5, length=max(lens))
    c.set_lengths(lens, [4] * B)
    q = torch.randn(B, Hq, 128, generator=torch.Generator().manual_seed(2)).cuda()
    res = {}
    for k in ("tc", "mma"):
        out = torch.zeros(B, Hq, 128, device="cuda")
        lse = torch.zeros(B, Hq, device="cuda")
        c.dense_decode_ex(0, q, out, None, 0, lse=lse, kernel=k)
        torch.cuda.synchronize()
        res[k] = (out, lse)
    assert rel_err(res["tc"][0].cpu().numpy(), res["mma"][0].cpu().numpy()) < 1e-4
    assert float((res["tc"][1] - res["mma"][1]).abs().max()) < 1e-4

"""Sequence sharding on one GPU: P shards driven in
lockstep by one process, the collectives emulated by plain tensor ops, against
the unsharded cache on the same rows:
  * dense / fast attention: LSE-merged partials within 2e-3 of the 1-GPU output;
  * pooled logits over each shard's J slice identical to the 1-GPU logits;
  * Selector indices (max / sums all-reduce, soft-NMS edges, top-k candidate
    merge) identical to the 1-GPU Selector on the same logits.
The CPU test runs the same exchange protocol over gloo (world 2 and 3) with a
numpy restatement of the decode Selector as the per-shard compute, against the
reference Selector.
"""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from helpers import oracle, rel_err

TOL = 2e-3


def _emulate(shards, attr, op):
    ts = [getattr(s, attr) for s in shards]
    if op == "max":
        r = torch.stack(ts).max(0).values
    elif op == "sum":
        r = torch.stack(ts).sum(0)
    for t in ts:
        t.copy_(r)


def _gather(shards, src, dst):
    g = torch.stack([getattr(s, src) for s in shards])
    for s in shards:
        getattr(s, dst).copy_(g.view_as(getattr(s, dst)))


def _selector(shards, layer, logits_of):
    for s in shards:
        s.sel_stats(layer, logits_of(s), 1)
    _emulate(shards, "row_max", "max")
    for s in shards:
        s.sel_stats(layer, logits_of(s), 2)
    _emulate(shards, "row_sums", "sum")
    for s in shards:
        s.sel_stats(layer, None, 3)
    _gather(shards, "edges", "edges_all")
    for s in shards:
        s.sel_finish(layer)
    _gather(shards, "cand_score", "cand_score_all")
    _gather(shards, "cand_pos", "cand_pos_all")
    for s in shards:
        s.sel_pick(layer)


def _partials(shards, outs):
    _gather(shards, "o_part", "o_all")
    _gather(shards, "lse_part", "lse_all")
    for s, o in zip(shards, outs):
        s.merge(o)


@pytest.mark.gpu
@pytest.mark.parametrize("P,H,Hq,prompt,K,B", [
    (2, 4, 64, 9000, 512, 1),    # C4 shape family: 4 KV heads, G = 16
    (4, 4, 16, 12000, 1024, 2),
    (3, 2, 4, 5000, 256, 1),     # uneven blocks
])
def test_sequence_sharded_step_matches_one_gpu(P, H, Hq, prompt, K, B):
    from paper_2603_12038_b200 import SelectorParams, SfiCache
    from paper_2603_12038_b200.sharded import SeqShardedSfi

    d, R, ns, Lmax = 128, 256, 4, prompt + 64
    full = SfiCache(1, B, H, Hq, d, Lmax, ns, K, R)
    full.fill_synthetic(seed=5, length=prompt)
    shards = [SeqShardedSfi(1, B, H, Hq, d, Lmax, prompt, ns, K, R, world=P, rank=r) for r in range(P)]
    for s in shards:
        n = min(s.cap, Lmax - s.base)
        s.k_cache[:, :, :, :n].copy_(full.k_cache[:, :, :, s.base:s.base + n])
        s.v_cache[:, :, :, :n].copy_(full.v_cache[:, :, :, s.base:s.base + n])
        s.key_norms[:, :, :, :n].copy_(full.key_norms[:, :, :, s.base:s.base + n])
        s.set_lengths([prompt] * B, [ns] * B)
    full.set_lengths([prompt] * B, [ns] * B)
    g = torch.Generator().manual_seed(P * 7 + H)
    q = torch.randn(B, Hq, d, generator=g).cuda()
    kn = torch.randn(B, H, d, generator=g).bfloat16().cuda()
    vn = torch.randn(B, H, d, generator=g).bfloat16().cuda()
    # ---- slow step: advance, append, dense (+ logits), Selector, compact ----
    full.step_advance()
    full.ring_append(0, kn, vn)
    for s in shards:
        s.step_advance()
        s.ring_append(0, kn, vn)
    out_full = torch.zeros(B, Hq, d, device="cuda")
    lg_full = torch.zeros_like(full.pooled_logits)
    full.dense_decode(0, q, out_full, lg_full, 0)
    full.selector(0, lg_full, SelectorParams())
    full.compact_build(0, rebuild_ring=True)
    lgs = [torch.zeros_like(s.pooled_logits) for s in shards]
    for s, lg in zip(shards, lgs):
        s.dense_partial(0, q, lg)
    outs = [torch.zeros(B, Hq, d, device="cuda") for _ in shards]
    _partials(shards, outs)
    torch.cuda.synchronize()
    full.check_errors()
    L = prompt + 1
    rl = min(R, L - ns)
    nJ = L - rl - ns
    for s, lg, o in zip(shards, lgs, outs):
        s.check_errors()
        assert rel_err(o.cpu().numpy(), out_full.cpu().numpy()) < TOL
        off, nloc = int(s.j_off[0]), int(s.prefix_len[0]) - int(s.n_sink_b[0]) - int(s.recent_len[0])
        assert int(s.n_glob[0]) == nJ
        if nloc > 0:  # the shard's J slice of the pooled logits
            assert torch.equal(lg[:, :, :nloc], lg_full[:, :, off:off + nloc])
    # Selector on each shard's own J slice of the (identical) pooled logits
    lg_of = {id(s): lg for s, lg in zip(shards, lgs)}
    _selector(shards, 0, lambda s: lg_of[id(s)])
    torch.cuda.synchronize()
    for b in range(B):
        for h in range(H):
            want = full.sel[0, b, h, : int(full.n_sel[0, b, h])].cpu()
            got = torch.cat([s.sel[0, b, h, : int(s.n_sel[0, b, h])].cpu() + s.base for s in shards])
            assert torch.equal(got, want), (b, h, len(got), len(want))
    for s in shards:
        s.compact_build(0, rebuild_ring=True)
    # ---- fast step: advance, fused append + sparse partials, merge ----
    full.step_advance()
    for s in shards:
        s.step_advance()
    kn2 = torch.randn(B, H, d, generator=g).bfloat16().cuda()
    full.fast_decode(0, q, kn2, kn2, out_full)
    for s in shards:
        s.fast_partial(0, q, kn2, kn2)
    _partials(shards, outs)
    torch.cuda.synchronize()
    full.check_errors()
    for s, o in zip(shards, outs):
        s.check_errors()
        assert rel_err(o.cpu().numpy(), out_full.cpu().numpy()) < TOL
    # the appended token lives on the last shard only, bit-identical
    last = shards[-1]
    Lg = L + 1
    assert torch.equal(last.k_cache[0, :, :, Lg - 1 - last.base].cpu(), full.k_cache[0, :, :, Lg - 1].cpu())
    assert torch.equal(last.key_norms[0, :, :, Lg - 1 - last.base].cpu(), full.key_norms[0, :, :, Lg - 1].cpu())

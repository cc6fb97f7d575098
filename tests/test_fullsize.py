"""Size-independent properties at BASELINE's full sizes (one layer of C2: 8
requests x 8 KV heads x 32K context, 32 q heads), where the CPU oracle would
take minutes: the compact gather is a bit-exact index gather of the paged cache;
full retention (every position of J selected) makes the fast step's sparse
attention equal the dense decode; the fused append writes exactly k_new/v_new."""
from __future__ import annotations

import numpy as np
import pytest

from helpers import rel_err

pytestmark = pytest.mark.gpu


def test_c2_full_retention_sparse_equals_dense_and_gather_bit_exact():
    import torch
    from paper_2603_12038_b200 import SfiCache

    B, H, Hq, d, ctx, ns, R = 8, 8, 32, 128, 32768, 4, 256
    nJ = ctx + 1 - R - ns  # |J| after the step advance
    c = SfiCache(1, B, H, Hq, d, ctx + 8, ns, nJ, R)  # k_budget = |J|: full retention
    c.fill_synthetic(seed=2028, length=ctx)
    c.set_lengths([ctx] * B, [ns] * B)
    c.step_advance()
    g = torch.Generator().manual_seed(1)
    kn = torch.randn(B, H, d, generator=g).bfloat16().cuda()
    c.ring_append(0, kn, kn)
    L = ctx + 1
    sel = torch.arange(ns + 1, L - R + 1, dtype=torch.int32, device="cuda")
    assert sel.numel() == nJ
    c.sel[0] = sel.expand(B, H, nJ)
    c.n_sel[0] = nJ
    c.compact_build(0, rebuild_ring=True)
    q = torch.randn(B, Hq, d, generator=g).cuda()
    out_d = torch.zeros_like(q)
    out_s = torch.zeros_like(q)
    c.dense_decode(0, q, out_d)
    c.sparse_decode(0, q, out_s)
    torch.cuda.synchronize()
    c.check_errors()
    # gather: compact rows R.. = paged rows of sink + selected, bit for bit
    idx = torch.cat([torch.arange(0, ns, device="cuda"), sel.long() - 1])
    assert torch.equal(c.ck[0, :, :, R:R + ns + nJ], c.k_cache[0][:, :, idx])
    assert torch.equal(c.cv[0, :, :, R:R + ns + nJ], c.v_cache[0][:, :, idx])
    # ring: slot (p - 1) % R holds position p for the last R positions
    pos = torch.arange(L - R + 1, L + 1, device="cuda")
    assert torch.equal(c.ck[0, :, :, (pos - 1) % R], c.k_cache[0][:, :, pos - 1])
    # full retention: support = all L positions -> sparse == dense (fp32 order only)
    assert rel_err(out_s.cpu().numpy(), out_d.cpu().numpy()) < 1e-4


def test_c2_fused_fast_step_append_full_size():
    import torch
    from paper_2603_12038_b200 import SelectorParams, SfiCache

    B, H, Hq, d, ctx = 8, 8, 32, 128, 32768
    c = SfiCache(1, B, H, Hq, d, ctx + 8, 4, 2048, 256)
    c.fill_synthetic(seed=2029, length=ctx)
    c.set_lengths([ctx] * B, [4] * B)
    q = torch.randn(B, Hq, d, generator=torch.Generator().manual_seed(3)).cuda()
    out = torch.zeros_like(q)
    lg = torch.zeros_like(c.pooled_logits)
    c.dense_decode(0, q, out, lg)
    c.selector(0, lg, SelectorParams())
    c.compact_build(0, rebuild_ring=True)
    c.step_advance()
    kn = torch.randn(B, H, d, generator=torch.Generator().manual_seed(4)).bfloat16().cuda()
    vn = torch.randn(B, H, d, generator=torch.Generator().manual_seed(5)).bfloat16().cuda()
    out_f = torch.zeros_like(q)
    c.fast_decode(0, q, kn, vn, out_f, prefetch=True)
    torch.cuda.synchronize()
    c.check_errors()
    L = ctx + 1
    assert torch.equal(c.k_cache[0, :, :, L - 1], kn) and torch.equal(c.v_cache[0, :, :, L - 1], vn)
    assert torch.equal(c.ck[0, :, :, (L - 1) % 256], kn) and torch.equal(c.cv[0, :, :, (L - 1) % 256], vn)
    # the same step through the unfused path on the same cache state
    out_u = torch.zeros_like(q)
    c.sparse_decode(0, q, out_u)
    torch.cuda.synchronize()
    assert rel_err(out_f.cpu().numpy(), out_u.cpu().numpy()) < 1e-4
    nrm = kn.double().pow(2).sum(-1).sqrt()
    assert np.allclose(c.key_norms[0, :, :, L - 1].cpu().numpy(), nrm.cpu().numpy(), rtol=1e-15)

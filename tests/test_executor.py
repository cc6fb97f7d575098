"""The C++ decode executor (include/sfi/decode.hpp) — the asynchronous slow step
(high-priority main stream, lowest-priority aux stream, pooled-logit slot ring,
one completion barrier) and the graph-captured step driven by
the device-resident per-step descriptor — replayed from its
CUDA graphs and checked against the CPU oracle layer by layer:

* slow step (graph replay): every layer's attention output vs the reference
  attention_kernel_dense (2e-3), its pooled logits (read from the executor's
  ring slot) vs the port's run_step capture (2e-3), the Selector's indices vs
  the reference run_selector on those logits (bit-exact), the compact gather vs
  the reference reorganize (bit-exact), the appended rows (bit-exact);
* the following fast step (graph replay): attention vs the reference
  attention_kernel_sparse on the selection just made (2e-3).
More layers than ring slots, so the slot back-pressure runs; inputs are views of
one packed [L][q | k | v] buffer (the bench's layout, non-default strides).
"""
from __future__ import annotations

import numpy as np
import pytest

from helpers import oracle, rel_err, store_from_rows

pytestmark = pytest.mark.gpu
TOL = 2e-3


def test_executor_graph_replayed_steps_match_oracle():
    import torch

    from oracle import oracle as O
    from paper_2603_12038_b200 import SfiCache
    from paper_2603_12038_b200.device import StepExecutor

    L, B, H, Hq, d, ns, K, R = 5, 2, 4, 16, 128, 4, 128, 64
    G = Hq // H
    lens = [3000, 2200]
    c = SfiCache(L, B, H, Hq, d, max(lens) + 8, ns, K, R)
    c.fill_synthetic(seed=41, length=max(lens))
    c.set_lengths(lens, [ns] * B)
    g = torch.Generator().manual_seed(8)
    qb, kb = B * Hq * d * 4, B * H * d * 2
    io = torch.empty(L, qb + 2 * kb, dtype=torch.uint8, device="cuda")
    q = io[:, :qb].view(torch.float32).view(L, B, Hq, d)
    kn = io[:, qb:qb + kb].view(torch.bfloat16).view(L, B, H, d)
    vn = io[:, qb + kb:].view(torch.bfloat16).view(L, B, H, d)
    q.copy_(torch.randn(L, B, Hq, d, generator=g))
    kn.copy_(torch.randn(L, B, H, d, generator=g).bfloat16())
    vn.copy_(torch.randn(L, B, H, d, generator=g).bfloat16())
    out = torch.zeros(L, B, Hq, d, device="cuda")
    torch.cuda.synchronize()
    x = StepExecutor(c, slots=2)  # 5 layers through 2 slots
    x.step(True, q, kn, vn, out, rebuild_ring=True)  # eager once (kernel attributes), then capture
    x.stream.synchronize()
    c.set_lengths(lens, [ns] * B)
    torch.cuda.synchronize()
    x.capture(True, q, kn, vn, out, rebuild_ring=True)
    out.zero_()
    x.replay(True)
    x.stream.synchronize()
    c.check_errors()
    ref, port = oracle("reference"), oracle("port")
    sink = list(range(1, ns + 1))
    for l in range(L):
        for b in range(B):
            Lb = int(c.prefix_len[b])
            rl = min(max(Lb - ns, 0), R)
            j0, j1 = ns + 1, Lb - rl
            assert torch.equal(c.k_cache[l, b, :, Lb - 1], kn[l, b]) and torch.equal(c.v_cache[l, b, :, Lb - 1], vn[l, b])
            k = c.k_cache[l, b, :, :Lb].float().cpu().numpy()
            v = c.v_cache[l, b, :, :Lb].float().cpu().numpy()
            st = store_from_rows(ref, k, v, Hq)
            want, _ = st.attention_dense(0, q[l, b].double().cpu().numpy())
            assert rel_err(out[l, b].cpu().numpy().reshape(-1), want) < TOL, (l, b)
            if l >= L - x.logits.shape[0]:  # the ring still holds the last `slots` layers' logits
                lg = x.logits_slot(l)[b, :, :j1 - j0 + 1].double().cpu().numpy()
                _, want_lg = store_from_rows(port, k, v, Hq).dense_capture(
                    0, q[l, b].double().cpu().numpy(), np.arange(j0, j1 + 1), 0)
                assert rel_err(lg, want_lg) < TOL, (l, b)
                norms = c.key_norms[l, b, :, j0 - 1:j1].cpu().numpy()
                want_sel, _ = ref.run_selector(lg, np.arange(j0, j1 + 1), norms, O.make_cfg(k_budget=K))
                for h in range(H):
                    got = c.sel[l, b, h, :int(c.n_sel[l, b, h])].cpu().numpy()
                    assert np.array_equal(got, want_sel[h]), (l, b, h)
            sel = [c.sel[l, b, h, :int(c.n_sel[l, b, h])].cpu().numpy() for h in range(H)]
            st.reorganize(0, sink, sel)
            for h in range(H):
                pos, rk, _ = st.compact(0, h)
                assert np.array_equal(c.ck[l, b, h, R:R + len(pos)].float().cpu().numpy(), rk), (l, b, h)
    # the next token: the fast step's graph
    q2 = torch.randn(L, B, Hq, d, generator=g).cuda()
    q.copy_(q2)
    x.step(False, q, kn, vn, out)  # eager once, then the same token again from the graph
    x.stream.synchronize()
    c.set_lengths([n + 1 for n in lens], [ns] * B)
    torch.cuda.synchronize()
    x.capture(False, q, kn, vn, out)
    out.zero_()
    x.replay(False)
    x.stream.synchronize()
    c.check_errors()
    for l in range(L):
        for b in range(B):
            Lb = int(c.prefix_len[b])
            rl = int(c.recent_len[b])
            k = c.k_cache[l, b, :, :Lb].float().cpu().numpy()
            v = c.v_cache[l, b, :, :Lb].float().cpu().numpy()
            st = store_from_rows(ref, k, v, Hq)
            sel = [c.sel[l, b, h, :int(c.n_sel[l, b, h])].cpu().numpy() for h in range(H)]
            st.reorganize(0, sink, sel)
            want, _ = st.attention_sparse(0, q[l, b].double().cpu().numpy(), sink, sel, Lb - rl + 1, rl)
            assert rel_err(out[l, b].cpu().numpy().reshape(-1), want) < TOL, ("fast", l, b)

"""Parity over a generation (C5's shape in miniature, BASELINE
configs[4]): a multi-step decode through the C++ executor's graph-replayed
steps, on the seeded slow / fast schedule (step 0 slow, triggers, forced at
t_max; scheduler.cpp:93-99), every step of every layer checked against the
reference on the cache state the device holds:

* each step: the appended row (bit-exact) and the attention output vs the
  reference attention_kernel_dense (slow) / attention_kernel_sparse on the
  current selection (fast), 2e-3;
* each slow step: the pooled logits vs the port's run_step capture (2e-3), the
  Selector's indices vs the reference run_selector on those logits
  (bit-exact), the compact gather vs the reference reorganize (bit-exact).
The selection carried into the fast steps is the one the device made and the
reference confirmed at the preceding slow step.
"""
from __future__ import annotations

import numpy as np
import pytest

from helpers import oracle, rel_err, store_from_rows

pytestmark = pytest.mark.gpu
TOL = 2e-3


def _schedule(n: int, t_max: int, p: float, seed: int) -> list[bool]:
    rng = np.random.default_rng(seed)
    out, since, trig = [], 0, True
    for _ in range(n):
        slow = trig or since + 1 >= t_max
        out.append(slow)
        since = 0 if slow else since + 1
        trig = bool(rng.random() < p)
    return out


def test_generation_parity_graph_replayed():
    import torch

    from oracle import oracle as O
    from paper_2603_12038_b200 import SfiCache
    from paper_2603_12038_b200.device import StepExecutor

    L, B, H, Hq, d, ns, K, R = 2, 2, 2, 8, 128, 4, 64, 32
    lens, n_steps = [900, 700], 36
    sched = _schedule(n_steps, t_max=8, p=1 / 6, seed=5)
    assert sum(sched) >= 4 and not all(sched)
    c = SfiCache(L, B, H, Hq, d, max(lens) + n_steps + 8, ns, K, R)
    c.fill_synthetic(seed=17, length=max(lens))
    c.set_lengths(lens, [ns] * B)
    q = torch.zeros(L, B, Hq, d, device="cuda")
    kn = torch.zeros(L, B, H, d, dtype=torch.bfloat16, device="cuda")
    vn = torch.zeros_like(kn)
    out = torch.zeros(L, B, Hq, d, device="cuda")
    x = StepExecutor(c, slots=2)
    g = torch.Generator().manual_seed(23)
    ref, port = oracle("reference"), oracle("port")
    sink = list(range(1, ns + 1))
    n_slow = 0
    for t, slow in enumerate(sched):
        q.copy_(torch.randn(L, B, Hq, d, generator=g))
        kn.copy_(torch.randn(L, B, H, d, generator=g).bfloat16())
        vn.copy_(torch.randn(L, B, H, d, generator=g).bfloat16())
        torch.cuda.synchronize()
        if t < 2:  # eager (the first slow step builds the ring), then both kinds captured once
            x.step(slow, q, kn, vn, out, rebuild_ring=(t == 0))
            x.stream.synchronize()
            if t == 1:
                pre = [int(v) for v in c.prefix_len.cpu()]
                for kind in (False, True):
                    x.capture(kind, q, kn, vn, out)
                assert [int(v) for v in c.prefix_len.cpu()] == pre  # capture does not run
        else:
            out.zero_()
            x.replay(slow)
            x.stream.synchronize()
        c.check_errors()
        n_slow += slow
        for l in range(L):
            for b in range(B):
                Lb = int(c.prefix_len[b])
                assert Lb == lens[b] + t + 1
                rl = min(max(Lb - ns, 0), R)
                assert int(c.recent_len[b]) == rl
                assert torch.equal(c.k_cache[l, b, :, Lb - 1], kn[l, b])
                assert torch.equal(c.v_cache[l, b, :, Lb - 1], vn[l, b])
                k = c.k_cache[l, b, :, :Lb].float().cpu().numpy()
                v = c.v_cache[l, b, :, :Lb].float().cpu().numpy()
                qd = q[l, b].double().cpu().numpy()
                st = store_from_rows(ref, k, v, Hq)
                sel = [c.sel[l, b, h, :int(c.n_sel[l, b, h])].cpu().numpy() for h in range(H)]
                if slow:
                    want, _ = st.attention_dense(0, qd)
                    assert rel_err(out[l, b].cpu().numpy().reshape(-1), want) < TOL, (t, l, b)
                    j0, j1 = ns + 1, Lb - rl
                    lg = x.logits_slot(l)[b, :, :j1 - j0 + 1].double().cpu().numpy()
                    _, want_lg = store_from_rows(port, k, v, Hq).dense_capture(0, qd, np.arange(j0, j1 + 1), 0)
                    assert rel_err(lg, want_lg) < TOL, (t, l, b)
                    norms = c.key_norms[l, b, :, j0 - 1:j1].cpu().numpy()
                    want_sel, _ = ref.run_selector(lg, np.arange(j0, j1 + 1), norms, O.make_cfg(k_budget=K))
                    for h in range(H):
                        assert np.array_equal(sel[h], want_sel[h]), (t, l, b, h)
                    st.reorganize(0, sink, sel)
                    for h in range(H):
                        pos, rk, _ = st.compact(0, h)
                        assert np.array_equal(c.ck[l, b, h, R:R + len(pos)].float().cpu().numpy(), rk), (t, l, b, h)
                else:
                    st.reorganize(0, sink, sel)
                    want, _ = st.attention_sparse(0, qd, sink, sel, Lb - rl + 1, rl)
                    assert rel_err(out[l, b].cpu().numpy().reshape(-1), want) < TOL, (t, l, b)
    assert n_slow == sum(sched)

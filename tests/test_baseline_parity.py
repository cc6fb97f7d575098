"""GPU parity at BASELINE.json's own sizes: one full layer of C2 (Qwen3-8B heads,
B = 8, 32K), C3 (Qwen3-32B heads, B = 4, 128K) and C4 (Qwen3-235B heads, B = 1,
256K) through the device path, checked against the CPU oracle on the identical
bf16 K/V, q and logits:

* K1 dense decode output vs the unmodified reference ``attention_kernel_dense``
  (oracle/_ref; attention.cpp:502-523), and vs the port's ``run_step`` capture
  restatement (bit-equal to the reference's attend, tests/test_oracle.py), whose
  pooled mean / max logits the device logits are compared with
  (attention.cpp:394-409) — within 2e-3 relative, max |got - want| / max |want|;
* K2 Selector indices bit-exact vs the reference ``run_selector`` on the device's
  own pooled logits and key norms (selector.cpp:254-299). At C3 and C4 |J| > 48K,
  so the 8-CTA cluster top-k runs (shared-memory keys at C3, global at C4);
* K3 compact gather bit-exact vs the reference ``KvStore::reorganize``/``compact``;
* K4 fused fast step (append + sparse) vs the reference ``attention_kernel_sparse``
  on the next token with the selection just made.

Every CTA of the stream-K dense grid streams 30+ tiles here (multi-tile online
softmax with lazy rescaling, slices split across CTAs and merged), and the K4
clusters 2-9 tiles per CTA. "peaked" inputs plant 32 high-affinity positions per
(b, KV head) with k = 3 q + N(0, 1), so the rescale branch runs and
the Selector sees structure; "iid" is N(0, 1) K/V with ragged lengths.

The CPU side runs one (request, KV head) unit per thread (ctypes drops the GIL);
a single-KV-head store performs exactly the per-head arithmetic of the full one
(attend walks one head's segments, attention.cpp:80-113, 258-268).
Set SFI_PARITY_REPORT=path to write the per-case error / mismatch figures.
"""
from __future__ import annotations

import concurrent.futures as cf
import json
import os
import subprocess
import sys

import numpy as np
import pytest

from helpers import oracle, rel_err, store_from_rows

pytestmark = pytest.mark.gpu

TOL = 2e-3
HERE = os.path.dirname(os.path.abspath(__file__))

CONFIGS = {  # SURVEY §8 shorthand table
    "C2": dict(B=8, H=8, Hq=32, ctx=32768),
    "C3": dict(B=4, H=8, Hq=64, ctx=131072),
    "C4": dict(B=1, H=4, Hq=64, ctx=262144),
}

_REPORT: dict = {}


def _workers() -> int:
    return max(1, min(32, os.cpu_count() or 1))


def _record(name, **kw):
    _REPORT[name] = kw
    path = os.environ.get("SFI_PARITY_REPORT")
    if path:
        os.makedirs(os.path.dirname(os.path.abspath(path)), exist_ok=True)
        with open(path, "w") as f:
            json.dump(_REPORT, f, indent=1, sort_keys=True)


def _layer_case(cfg: str, inputs: str, pool: int, seed: int):
    import torch

    from paper_2603_12038_b200 import SelectorParams, SfiCache

    p = CONFIGS[cfg]
    B, H, Hq, ctx, d, ns, K, R = p["B"], p["H"], p["Hq"], p["ctx"], 128, 4, 2048, 256
    G = Hq // H
    lens = [ctx - (1000 * b if inputs == "iid" else 0) for b in range(B)]
    c = SfiCache(1, B, H, Hq, d, ctx + 8, ns, K, R)
    c.fill_synthetic(seed=seed, length=ctx)
    c.set_lengths(lens, [ns] * B)
    g = torch.Generator().manual_seed(seed)
    q = torch.randn(B, Hq, d, generator=g)
    if inputs == "peaked":
        c.plant_peaked(0, q.cuda(), n_planted=32, scale=3.0, seed=seed)
    # one decode step: append the current token, dense decode + capture, Selector, compact
    c.step_advance()
    kn = torch.randn(B, H, d, generator=g).bfloat16()
    vn = torch.randn(B, H, d, generator=g).bfloat16()
    c.ring_append(0, kn.cuda(), vn.cuda())
    out = torch.zeros(B, Hq, d, device="cuda")
    logits = torch.zeros_like(c.pooled_logits)
    c.dense_decode(0, q.cuda(), out, logits, pool)
    out_share = torch.zeros_like(out)
    c.dense_decode_ex(0, q.cuda(), out_share, None, pool, share_sm=True)  # the timed slow step's grid
    c.selector(0, logits, SelectorParams())
    c.compact_build(0, rebuild_ring=True)
    torch.cuda.synchronize()
    c.check_errors()
    # next token: the fused fast step (K4) on the selection just made
    c.step_advance()
    kn2 = torch.randn(B, H, d, generator=g).bfloat16()
    vn2 = torch.randn(B, H, d, generator=g).bfloat16()
    q2 = torch.randn(B, Hq, d, generator=g)
    out_f = torch.zeros(B, Hq, d, device="cuda")
    c.fast_decode(0, q2.cuda(), kn2.cuda(), vn2.cuda(), out_f, prefetch=True)
    torch.cuda.synchronize()
    c.check_errors()

    L1 = [int(x) for x in (c.prefix_len - 1).cpu()]          # slow-step context per request
    rl1 = [min(max(L - ns, 0), R) for L in L1]                 # its recent window (scheduler.cpp:45-51)
    L2 = [int(x) for x in c.prefix_len.cpu()]
    rl2 = [int(x) for x in c.recent_len.cpu()]
    out = out.cpu().numpy()
    out_share = out_share.cpu().numpy()
    out_f = out_f.cpu().numpy()
    sel = c.sel[0].cpu().numpy()
    n_sel = c.n_sel[0].cpu().numpy()
    ck = c.ck[0].float().cpu().numpy()
    cvv = c.cv[0].float().cpu().numpy()
    ref, port = oracle("reference"), oracle("port")
    from oracle import oracle as O

    # ---- Selector, one request per unit (cross-head couples the heads) ----
    def selector_unit(b):
        j0, j1 = ns + 1, L1[b] - rl1[b]
        n = j1 - j0 + 1
        vals = logits[b, :, :n].double().cpu().numpy()
        norms = c.key_norms[0, b, :, j0 - 1:j1].cpu().numpy()
        want, _ = ref.run_selector(vals, np.arange(j0, j1 + 1), norms, O.make_cfg(k_budget=K, pool=pool))
        mism = 0
        for h in range(H):
            got = sel[b, h, :n_sel[b, h]]
            if not np.array_equal(got, want[h]):
                mism += 1 + int(np.setxor1d(got, want[h]).size)
        return want, mism, n

    # ---- attention, one (request, KV head) unit per thread ----
    def attn_unit(bh):
        b, h = bh
        Lb = L2[b]
        k = c.k_cache[0, b, h:h + 1, :Lb].float().cpu().numpy()
        v = c.v_cache[0, b, h:h + 1, :Lb].float().cpu().numpy()
        qs = q[b, h * G:(h + 1) * G].double().numpy()
        q2s = q2[b, h * G:(h + 1) * G].double().numpy()
        st_r = store_from_rows(ref, k[:, :L1[b]], v[:, :L1[b]], G)
        st_p = store_from_rows(port, k[:, :L1[b]], v[:, :L1[b]], G)
        j0, j1 = ns + 1, L1[b] - rl1[b]
        want_o, _ = st_r.attention_dense(0, qs)
        cap_o, cap_lg = st_p.dense_capture(0, qs, np.arange(j0, j1 + 1), pool)
        assert np.array_equal(want_o, cap_o), "port capture output != reference attend"
        got_o = out[b, h * G:(h + 1) * G].reshape(-1)
        got_s = out_share[b, h * G:(h + 1) * G].reshape(-1)
        got_lg = logits[b, h, :j1 - j0 + 1].cpu().numpy()
        e_dense = max(rel_err(got_o, want_o), rel_err(got_s, want_o))
        e_lg = rel_err(got_lg, cap_lg[0])
        # compact gather + the fused fast step on the next token
        sink = list(range(1, ns + 1))
        selh = [sel[b, h, :n_sel[b, h]].astype(np.int32)]
        st_r.append_many(k[0, L1[b]:L2[b]].reshape(-1, 128), v[0, L1[b]:L2[b]].reshape(-1, 128))
        st_r.reorganize(0, sink, selh)
        pos, rk, rv = st_r.compact(0, 0)
        gather_ok = (np.array_equal(ck[b, h, R:R + len(pos)], rk) and np.array_equal(cvv[b, h, R:R + len(pos)], rv))
        want_f, _ = st_r.attention_sparse(0, q2s, sink, selh, L2[b] - rl2[b] + 1, rl2[b])
        e_fast = rel_err(out_f[b, h * G:(h + 1) * G].reshape(-1), want_f)
        return e_dense, e_lg, gather_ok, e_fast

    with cf.ThreadPoolExecutor(_workers()) as ex:
        sel_f = [ex.submit(selector_unit, b) for b in range(B)]
        att = list(ex.map(attn_unit, [(b, h) for b in range(B) for h in range(H)]))
        sel_r = [f.result() for f in sel_f]
    # the appended rows are the tokens written, bit for bit
    for b in range(B):
        assert torch.equal(c.k_cache[0, b, :, L1[b] - 1].cpu(), kn[b])
        assert torch.equal(c.k_cache[0, b, :, L2[b] - 1].cpu(), kn2[b])
    res = dict(
        dense_rel_err=max(a[0] for a in att), logit_rel_err=max(a[1] for a in att),
        gather_bit_exact=all(a[2] for a in att), fast_rel_err=max(a[3] for a in att),
        selector_mismatched_positions=sum(s[1] for s in sel_r), selector_rows=B * H,
        n_J=[s[2] for s in sel_r], context=L1, pool=["mean", "max"][pool], inputs=inputs)
    _record(f"{cfg}_{inputs}_{res['pool']}", **res)
    return res


@pytest.mark.parametrize("cfg,inputs,pool,seed", [
    ("C2", "iid", 0, 2027),
    ("C2", "peaked", 1, 2127),
    ("C3", "peaked", 0, 2028),
    ("C4", "peaked", 0, 2029),
    ("C4", "iid", 1, 2129),
])
def test_full_layer_parity(cfg, inputs, pool, seed):
    if not oracle().kind == "reference":
        pytest.skip("oracle/_ref not built")
    r = _layer_case(cfg, inputs, pool, seed)
    assert r["selector_mismatched_positions"] == 0, r
    assert r["gather_bit_exact"], r
    assert r["dense_rel_err"] < TOL and r["logit_rel_err"] < TOL and r["fast_rel_err"] < TOL, r


# ---- exact ties across the decode Selector's statistics chunks (512 positions) ----

@pytest.mark.parametrize("refine", [False, True])
def test_selector_exact_ties_across_chunks(refine):
    """Logits quantized to a few levels and repeated in every 512-position chunk,
    lambda_clip = 0 (s = f exactly): hundreds of exactly tied scores straddle the
    K-th place; the reference resolves them to the lower position (selector.cpp:
    243-247) and so must the device (p from the row max, not a chunk max)."""
    import torch

    from oracle import oracle as O
    from paper_2603_12038_b200 import SelectorConfig, SelectorParams, SfiCache

    B, H, Hq, ctx, ns, K, R = 2, 4, 8, 6000, 4, 256, 64
    c = SfiCache(1, B, H, Hq, 128, ctx + 8, ns, K, R)
    c.fill_synthetic(seed=5, length=ctx)
    c.set_lengths([ctx, ctx - 1700], [ns] * B)
    rng = np.random.default_rng(3)
    base = np.round(rng.normal(0, 1, size=(H, 512)) * 2) / 2          # a few levels per head
    lg = np.tile(base, (1, (ctx + 8 + 511) // 512))[:, :ctx + 8]         # repeated in every chunk
    logits = torch.from_numpy(np.broadcast_to(lg, (B, H, ctx + 8)).astype(np.float32).copy()).cuda()
    cfg = SelectorConfig()
    cfg.k_budget = K
    kw = dict(lambda_clip=0.0)
    if not refine:
        kw.update(alpha_soft=0.0, alpha_cross=0.0)
    for k_, v_ in kw.items():
        setattr(cfg, k_, v_)
    c.selector(0, logits, SelectorParams(cfg))
    torch.cuda.synchronize()
    c.check_errors()
    for b in range(B):
        L, rl = int(c.prefix_len[b]), int(c.recent_len[b])
        j0, j1 = ns + 1, L - rl
        n = j1 - j0 + 1
        vals = logits[b, :, :n].double().cpu().numpy()
        norms = c.key_norms[0, b, :, j0 - 1:j1].cpu().numpy()
        want, st = oracle().run_selector(vals, np.arange(j0, j1 + 1), norms, O.make_cfg(k_budget=K, **kw),
                                         stages=True)
        for h in range(H):
            z = st["z_adj"][h]
            kth = np.sort(z)[::-1][K - 1]
            if not refine:
                assert (z == kth).sum() > 1, "the case must put exact ties at the K-th place"
            got = c.sel[0, b, h, :int(c.n_sel[0, b, h])].cpu().numpy()
            assert np.array_equal(got, want[h]), (b, h)


# ---- the cluster top-k variants forced at small sizes (SFI_TOPK_CLUSTER) ----

@pytest.mark.parametrize("force", ["cluster=1", "cluster=4", "bt=1"])
def test_forced_cluster_topk(force):
    """The top-k variant is chosen per process from the environment: run the
    Selector parity check in a child with it forced — SFI_TOPK_CLUSTER (8-CTA or
    4-CTA clusters, shared-memory keys at |J| = 5K, global keys at |J| = 100K with
    4 CTAs) or SFI_TOPK_BT (the long-row histogram top-k at both lengths)."""
    kind, val = force.split("=")
    env = dict(os.environ, **{"SFI_TOPK_CLUSTER" if kind == "cluster" else "SFI_TOPK_BT": val})
    r = subprocess.run([sys.executable, os.path.join(HERE, "_topk_cluster_case.py")], env=env,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    assert "ok" in r.stdout


@pytest.mark.parametrize("refine", [False, True])
def test_long_row_topk_exact_ties(refine):
    """The long-row top-k (|J| > 48K: value histogram + listed threshold bin, rows x
    segments) with massive exact ties straddling the K-th place (quantized logits
    repeated in every chunk, lambda_clip = 0): indices equal the reference's."""
    import torch

    from oracle import oracle as O
    from paper_2603_12038_b200 import SelectorConfig, SelectorParams, SfiCache

    B, H, Hq, ctx, ns, K, R = 1, 4, 8, 60000, 4, 2048, 64
    c = SfiCache(1, B, H, Hq, 128, ctx + 8, ns, K, R)
    c.fill_synthetic(seed=6, length=ctx)
    c.set_lengths([ctx], [ns])
    rng = np.random.default_rng(9)
    base = np.round(rng.normal(0, 1, size=(H, 512)) * 2) / 2
    lg = np.tile(base, (1, (ctx + 8 + 511) // 512))[:, :ctx + 8]
    logits = torch.from_numpy(np.broadcast_to(lg, (B, H, ctx + 8)).astype(np.float32).copy()).cuda()
    cfg = SelectorConfig()
    cfg.k_budget = K
    kw = dict(lambda_clip=0.0) if refine else dict(lambda_clip=0.0, alpha_soft=0.0, alpha_cross=0.0)
    for k_, v_ in kw.items():
        setattr(cfg, k_, v_)
    c.selector(0, logits, SelectorParams(cfg))
    torch.cuda.synchronize()
    c.check_errors()
    L, rl = int(c.prefix_len[0]), int(c.recent_len[0])
    j0, j1 = ns + 1, L - rl
    vals = logits[0, :, :j1 - j0 + 1].double().cpu().numpy()
    norms = c.key_norms[0, 0, :, j0 - 1:j1].cpu().numpy()
    want, _ = oracle().run_selector(vals, np.arange(j0, j1 + 1), norms, O.make_cfg(k_budget=K, **kw))
    for h in range(H):
        got = c.sel[0, 0, h, :int(c.n_sel[0, 0, h])].cpu().numpy()
        assert np.array_equal(got, want[h]), h


def test_long_row_topk_ragged_batch():
    """The long-row top-k over a ragged batch (rows of different |J| in one launch,
    one row with |J| <= K that takes all of J, one empty J) on peaked inputs: every
    row's indices equal the reference's run_selector on the device's logits."""
    import torch

    from oracle import oracle as O
    from paper_2603_12038_b200 import SelectorParams, SfiCache

    H, Hq, ns, K, R = 2, 8, 4, 2048, 64
    lens = [70000, 49500, 1900, 40]
    B = len(lens)
    c = SfiCache(1, B, H, Hq, 128, max(lens) + 8, ns, K, R)
    c.fill_synthetic(seed=12, length=max(lens))
    c.set_lengths(lens, [ns] * B)
    q = torch.randn(B, Hq, 128, generator=torch.Generator().manual_seed(12)).cuda()
    c.plant_peaked(0, q, n_planted=32, scale=3.0, seed=12)
    out = torch.zeros_like(q)
    logits = torch.zeros_like(c.pooled_logits)
    c.dense_decode(0, q, out, logits, 0)
    c.selector(0, logits, SelectorParams())
    torch.cuda.synchronize()
    c.check_errors()
    ref = oracle()
    for b in range(B):
        L, rl = int(c.prefix_len[b]), int(c.recent_len[b])
        j0, j1 = ns + 1, L - rl
        if j1 < j0:  # empty J: no selection
            assert all(int(c.n_sel[0, b, h]) == 0 for h in range(H)), b
            continue
        vals = logits[b, :, :j1 - j0 + 1].double().cpu().numpy()
        norms = c.key_norms[0, b, :, j0 - 1:j1].cpu().numpy()
        want, _ = ref.run_selector(vals, np.arange(j0, j1 + 1), norms, O.make_cfg(k_budget=K))
        for h in range(H):
            got = c.sel[0, b, h, :int(c.n_sel[0, b, h])].cpu().numpy()
            assert np.array_equal(got, want[h]), (b, h)


def test_long_row_topk_nondefault_config():
    """The long-row top-k with a non-default Selector config (stronger soft-NMS and
    cross-head terms, temperature != 1, radius 3, wider lambda clip, other prior
    exponent): the histogram's value range follows alpha_soft / alpha_cross, and
    the indices equal the reference's."""
    import torch

    from oracle import oracle as O
    from paper_2603_12038_b200 import SelectorConfig, SelectorParams, SfiCache

    B, H, Hq, ctx, ns, K, R = 1, 4, 16, 66000, 4, 1500, 128
    c = SfiCache(1, B, H, Hq, 128, ctx + 8, ns, K, R)
    c.fill_synthetic(seed=21, length=ctx)
    c.set_lengths([ctx], [ns])
    q = torch.randn(B, Hq, 128, generator=torch.Generator().manual_seed(21)).cuda()
    c.plant_peaked(0, q, n_planted=32, scale=3.0, seed=21)
    out = torch.zeros_like(q)
    logits = torch.zeros_like(c.pooled_logits)
    c.dense_decode(0, q, out, logits, 0)
    kw = dict(alpha_soft=0.8, alpha_cross=0.6, temperature=0.7, nms_radius=3, lambda_clip=0.05, beta=2.0)
    cfg = SelectorConfig()
    cfg.k_budget = K
    for k_, v_ in kw.items():
        setattr(cfg, k_, v_)
    c.selector(0, logits, SelectorParams(cfg))
    torch.cuda.synchronize()
    c.check_errors()
    L, rl = int(c.prefix_len[0]), int(c.recent_len[0])
    j0, j1 = ns + 1, L - rl
    vals = logits[0, :, :j1 - j0 + 1].double().cpu().numpy()
    norms = c.key_norms[0, 0, :, j0 - 1:j1].cpu().numpy()
    want, _ = oracle().run_selector(vals, np.arange(j0, j1 + 1), norms, O.make_cfg(k_budget=K, **kw))
    for h in range(H):
        got = c.sel[0, 0, h, :int(c.n_sel[0, 0, h])].cpu().numpy()
        assert np.array_equal(got, want[h]), h

"""Sequence sharding on one GPU: P shards driven in
lockstep by one process, the collectives emulated by plain tensor ops, against
the unsharded cache on the same rows:
  * dense / fast attention: LSE-merged partials within 2e-3 of the 1-GPU output;
  * pooled logits over each shard's J slice identical to the 1-GPU logits;
  * Selector indices (max / sums all-reduce, soft-NMS edges, top-k candidate
    merge) identical to the 1-GPU Selector on the same logits.
The CPU test runs the same exchange protocol over gloo (world 2 and 3) with a
numpy restatement of the decode Selector as the per-shard compute, against the
reference Selector: local statistics -> all-gather -> global rescale, soft-NMS
edges -> all-gather, top-k candidates -> all-gather -> pick.
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


def _gather(shards, src, dst):
    g = torch.stack([getattr(s, src) for s in shards])
    for s in shards:
        getattr(s, dst).copy_(g.view_as(getattr(s, dst)))


def _selector(shards, layer, logits_of):
    for s in shards:
        s.sel_stats(layer, logits_of(s), 1)
    _gather(shards, "row_stats", "stats_all")
    for s in shards:
        s.sel_stats(layer, logits_of(s), 3)
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


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _seq_gpu_worker(rank, world, port, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        from paper_2603_12038_b200 import SelectorParams, SfiCache
        from paper_2603_12038_b200.sharded import SeqShardedSfi

        B, H, Hq, d, prompt, K, R, ns = 1, 4, 64, 128, 6000, 256, 256, 4
        Lmax = prompt + 16
        full = SfiCache(1, B, H, Hq, d, Lmax, ns, K, R)
        full.fill_synthetic(seed=3, length=prompt)  # identical on every rank
        sh = SeqShardedSfi(1, B, H, Hq, d, Lmax, prompt, ns, K, R)
        n = min(sh.cap, Lmax - sh.base)
        sh.k_cache[:, :, :, :n].copy_(full.k_cache[:, :, :, sh.base:sh.base + n])
        sh.v_cache[:, :, :, :n].copy_(full.v_cache[:, :, :, sh.base:sh.base + n])
        sh.key_norms[:, :, :, :n].copy_(full.key_norms[:, :, :, sh.base:sh.base + n])
        sh.set_lengths([prompt], [ns])
        full.set_lengths([prompt], [ns])
        g = torch.Generator().manual_seed(8)
        qv = torch.randn(B, Hq, d, generator=g).cuda()
        kn = torch.randn(B, H, d, generator=g).bfloat16().cuda()
        ok = True
        for step, slow in enumerate((True, False, False)):
            full.step_advance()
            sh.step_advance()
            o_full = torch.zeros(B, Hq, d, device="cuda")
            o_sh = torch.zeros_like(o_full)
            if slow:
                full.ring_append(0, kn, kn)
                sh.ring_append(0, kn, kn)
                lg_f, lg_s = torch.zeros_like(full.pooled_logits), torch.zeros_like(sh.pooled_logits)
                full.dense_decode(0, qv, o_full, lg_f, 0)
                full.selector(0, lg_f, SelectorParams())
                full.compact_build(0, rebuild_ring=True)
                sh.dense_decode(0, qv, o_sh, lg_s, 0)
                sh.selector(0, lg_s)
                sh.compact_build(0, rebuild_ring=True)
                torch.cuda.synchronize()
                sel = [torch.zeros(B, H, K, dtype=torch.int32) for _ in range(world)]
                cnt = [torch.zeros(B, H, dtype=torch.int32) for _ in range(world)]
                dist.all_gather(sel, sh.sel[0].cpu())
                dist.all_gather(cnt, sh.n_sel[0].cpu())
                for h in range(H):
                    got = torch.cat([sel[r][0, h, : int(cnt[r][0, h])] + r * sh.block for r in range(world)])
                    ok &= torch.equal(got, full.sel[0, 0, h, : int(full.n_sel[0, 0, h])].cpu())
            else:
                full.fast_decode(0, qv, kn, kn, o_full)
                sh.fast_decode(0, qv, kn, kn, o_sh)
            torch.cuda.synchronize()
            full.check_errors()
            sh.check_errors()
            ok &= rel_err(o_sh.cpu().numpy(), o_full.cpu().numpy()) < TOL
        q.put((rank, bool(ok)))
        dist.destroy_process_group()
    except Exception:  # pragma: no cover
        import traceback

        q.put((rank, traceback.format_exc()))


@pytest.mark.gpu
def test_sequence_sharded_two_processes_one_gpu():
    ctx = mp.get_context("spawn")
    qu = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_seq_gpu_worker, args=(r, 2, port, qu)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(qu.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {0: True, 1: True}, res


@pytest.mark.gpu
@pytest.mark.parametrize("P", [2, 3])
def test_sequence_sharded_peer_exchange_lockstep(P):
    """Peer-memory (O, LSE) exchange (sfi_peer_publish / sfi_peer_merge) over 2 layers
    and 3 steps: bit-identical to merging gathered copies, within 2e-3 of 1 GPU."""
    from paper_2603_12038_b200 import SelectorParams, SfiCache
    from paper_2603_12038_b200.sharded import SeqShardedSfi, connect_lockstep

    B, H, Hq, d, prompt, K, R, ns, NL = 1, 4, 16, 128, 7000, 256, 256, 4, 2
    Lmax = prompt + 16
    full = SfiCache(NL, B, H, Hq, d, Lmax, ns, K, R)
    full.fill_synthetic(seed=9, length=prompt)
    shards = [SeqShardedSfi(NL, B, H, Hq, d, Lmax, prompt, ns, K, R, world=P, rank=r, peers=[]) for r in range(P)]
    connect_lockstep(shards)
    for s in shards:
        n = min(s.cap, Lmax - s.base)
        s.k_cache[:, :, :, :n].copy_(full.k_cache[:, :, :, s.base:s.base + n])
        s.v_cache[:, :, :, :n].copy_(full.v_cache[:, :, :, s.base:s.base + n])
        s.key_norms[:, :, :, :n].copy_(full.key_norms[:, :, :, s.base:s.base + n])
        s.set_lengths([prompt] * B, [ns] * B)
    full.set_lengths([prompt] * B, [ns] * B)
    g = torch.Generator().manual_seed(P)
    for step, slow in enumerate((True, False, False)):
        full.step_advance()
        for s in shards:
            s.step_advance()
        for layer in range(NL):
            q = torch.randn(B, Hq, d, generator=g).cuda()
            kn = torch.randn(B, H, d, generator=g).bfloat16().cuda()
            o_full = torch.zeros(B, Hq, d, device="cuda")
            outs = [torch.zeros_like(o_full) for _ in shards]
            if slow:
                full.ring_append(layer, kn, kn)
                lg_full = torch.zeros_like(full.pooled_logits)
                full.dense_decode(layer, q, o_full, lg_full, 0)
                full.selector(layer, lg_full, SelectorParams())
                full.compact_build(layer, rebuild_ring=True)
                lgs = [torch.zeros_like(s.pooled_logits) for s in shards]
                for s, lg in zip(shards, lgs):
                    s.ring_append(layer, kn, kn)
                    s.dense_partial(layer, q, lg)  # + publish
            else:
                full.fast_decode(layer, q, kn, kn, o_full)
                for s in shards:
                    s.fast_partial(layer, q, kn, kn)  # + publish
            for s, o in zip(shards, outs):
                s.peer_merge(layer, o)
            # the same partials through the gather path
            slot = layer % shards[0].px.slots
            o_all = torch.stack([s.px.o[slot] for s in shards]).contiguous()
            lse_all = torch.stack([s.px.lse[slot] for s in shards]).contiguous()
            ref = torch.zeros_like(o_full)
            shards[0]._C.merge_partials(P, B * Hq, d, o_all.data_ptr(), lse_all.data_ptr(), ref.data_ptr(),
                                        torch.cuda.current_stream().cuda_stream)
            torch.cuda.synchronize()
            for o in outs:
                assert torch.equal(o, ref), (step, layer)
                assert rel_err(o.cpu().numpy(), o_full.cpu().numpy()) < TOL, (step, layer)
            if slow:  # the Selector's three exchanges over peer memory, in lockstep
                st = torch.cuda.current_stream().cuda_stream
                for s, lg in zip(shards, lgs):
                    s.sel_stats(layer, lg, 1)
                    s.px.publish(st)
                for s in shards:
                    s.px.gather("row_stats", s.stats_all, st)
                for s, lg in zip(shards, lgs):
                    s.sel_stats(layer, lg, 3)
                    s.px.publish(st)
                for s in shards:
                    s.px.gather("edges", s.edges_all, st)
                for s in shards:
                    s.sel_finish(layer)
                    s.px.publish(st)
                for s in shards:
                    s.px.gather("cand_score", s.cand_score_all, st)
                    s.px.gather("cand_pos", s.cand_pos_all, st)
                    s.sel_pick(layer)
                torch.cuda.synchronize()
                for b in range(B):
                    for h in range(H):
                        want = full.sel[layer, b, h, : int(full.n_sel[layer, b, h])].cpu()
                        got = torch.cat([s.sel[layer, b, h, : int(s.n_sel[layer, b, h])].cpu() + s.base
                                         for s in shards])
                        assert torch.equal(got, want), (layer, b, h)
                for s in shards:
                    s.compact_build(layer, rebuild_ring=True)
    for s in shards:
        s.check_errors()
    assert all(int(s.px.flag[0]) == 3 * NL + 3 * NL for s in shards)  # partials + Selector exchanges


def _seq_peer_worker(rank, world, port, q):
    """Two processes on one GPU: partials exchanged through CUDA IPC mappings
    (PeerExchange), against the gather path in the same process and 1 GPU."""
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        from paper_2603_12038_b200 import SelectorParams, SfiCache
        from paper_2603_12038_b200.sharded import SeqShardedSfi

        B, H, Hq, d, prompt, K, R, ns, NL = 1, 4, 16, 128, 6000, 256, 256, 4, 2
        Lmax = prompt + 16
        full = SfiCache(NL, B, H, Hq, d, Lmax, ns, K, R)
        full.fill_synthetic(seed=3, length=prompt)  # identical on every rank
        shp = SeqShardedSfi(NL, B, H, Hq, d, Lmax, prompt, ns, K, R, peer=True)
        shg = SeqShardedSfi(NL, B, H, Hq, d, Lmax, prompt, ns, K, R)
        for sh in (shp, shg):
            n = min(sh.cap, Lmax - sh.base)
            sh.k_cache[:, :, :, :n].copy_(full.k_cache[:, :, :, sh.base:sh.base + n])
            sh.v_cache[:, :, :, :n].copy_(full.v_cache[:, :, :, sh.base:sh.base + n])
            sh.key_norms[:, :, :, :n].copy_(full.key_norms[:, :, :, sh.base:sh.base + n])
            sh.set_lengths([prompt], [ns])
        full.set_lengths([prompt], [ns])
        g = torch.Generator().manual_seed(8)
        ok = True
        for step in range(3):
            full.step_advance()
            for sh in (shp, shg):
                sh.step_advance()
            for layer in range(NL):
                qv = torch.randn(B, Hq, d, generator=g).cuda()
                kn = torch.randn(B, H, d, generator=g).bfloat16().cuda()
                o_full, o_p, o_g = (torch.zeros(B, Hq, d, device="cuda") for _ in range(3))
                full.ring_append(layer, kn, kn)
                lg_f = torch.zeros_like(full.pooled_logits)
                full.dense_decode(layer, qv, o_full, lg_f, 0)
                full.selector(layer, lg_f, SelectorParams())
                sels = []
                for sh, o in ((shp, o_p), (shg, o_g)):
                    sh.ring_append(layer, kn, kn)
                    lg = torch.zeros_like(sh.pooled_logits)
                    sh.dense_decode(layer, qv, o, lg, 0)
                    sh.selector(layer, lg)  # peer-memory exchanges for shp, all-gathers for shg
                    sels.append((sh.sel[layer].clone(), sh.n_sel[layer].clone()))
                torch.cuda.synchronize()
                ok &= torch.equal(o_p, o_g)
                ok &= rel_err(o_p.cpu().numpy(), o_full.cpu().numpy()) < TOL
                ok &= torch.equal(sels[0][0], sels[1][0]) and torch.equal(sels[0][1], sels[1][1])
        full.check_errors()
        shp.check_errors()
        q.put((rank, bool(ok)))
        dist.barrier()
        dist.destroy_process_group()
    except Exception:  # pragma: no cover
        import traceback

        q.put((rank, traceback.format_exc()))


@pytest.mark.gpu
def test_sequence_sharded_peer_exchange_two_processes_one_gpu():
    ctx = mp.get_context("spawn")
    qu = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_seq_peer_worker, args=(r, 2, port, qu)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(qu.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {0: True, 1: True}, res


# ------------------------------------------------------------- CPU, gloo ----

def _np_case(seed=4, H=4, n=2500):
    rng = np.random.default_rng(seed)
    vals = rng.normal(0.0, 0.4, size=(H, n))
    norms = np.abs(rng.normal(11.0, 2.0, size=(H, n))) + 0.1
    return vals, norms, np.arange(5, 5 + n, dtype=np.int32)


def _seq_protocol_worker(rank, world, port, cuts, q):
    """The device protocol of sequence-sharded Selector (sharded.py
    SeqShardedSfi.selector), with a numpy restatement of the per-shard stages
    (selector.cu decode fast path) and the real gloo collectives."""
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from oracle import oracle as O
        from paper_2603_12038_b200.sharded import all_gather_blocks

        vals, norms, allowed = _np_case()
        H, ng = vals.shape
        K, R, eps = 300, 2, 1e-8
        a, b = cuts[rank], cuts[rank + 1]
        v, nm, n = vals[:, a:b], norms[:, a:b], b - a
        # phase 1: local max (from kMaskedLogit) and the five sums relative to it
        ml = np.maximum(v.max(1) if n else -1e30, -1e30).astype(np.float64)
        u = (np.arange(a, b) / ((ng - 1) + eps))[None, :]
        pl = np.exp(v - ml[:, None])
        w = (1.0 / (nm + eps)) * np.exp(-(u * u)) * np.sqrt(1.0 - u + eps)
        st = np.stack([ml, pl.sum(1), w.sum(1), (pl * pl).sum(1), (pl * w).sum(1), (w * w).sum(1)], 1)
        stats_all = torch.zeros(world, H, 6, dtype=torch.float64)
        all_gather_blocks(torch.from_numpy(st), stats_all)
        # combine in shard order, rescaled to the global max
        SA = stats_all.numpy()
        M = SA[:, :, 0].max(0)
        e = np.exp(SA[:, :, 0] - M[None, :])
        S = np.stack([(SA[:, :, 1] * e).sum(0), SA[:, :, 2].sum(0), (SA[:, :, 3] * e * e).sum(0),
                      (SA[:, :, 4] * e).sum(0), SA[:, :, 5].sum(0)], 1)
        p = np.exp(v - M[:, None])  # phase 3 recomputes p against the global max
        c1, c2 = 1.0 / S[:, 0], 1.0 / S[:, 1]
        ff, fr, rr = S[:, 2] * c1 * c1, S[:, 3] * c1 * c2, S[:, 4] * c2 * c2
        den = ff - 2 * fr + rr
        lam = np.where(np.abs(den) >= eps, np.clip((ff - fr) / np.where(den == 0, 1, den), 0, 0.02), 0.0)
        z = np.log((1 - lam)[:, None] * c1[:, None] * p + lam[:, None] * c2[:, None] * w + eps)
        # phase 3: edges (first R, last R, j_off, n), all-gather
        nan = float("nan")
        edge = np.full((H, 2 * R + 2), nan)
        for h in range(H):
            for t in range(R):
                if t < n:
                    edge[h, t] = z[h, t]
                if 0 <= n - R + t < n:
                    edge[h, R + t] = z[h, n - R + t]
            edge[h, 2 * R], edge[h, 2 * R + 1] = a, n
        edges = torch.zeros(world, H, 2 * R + 2, dtype=torch.float64)
        all_gather_blocks(torch.from_numpy(edge), edges)
        E = edges.numpy()

        def zg(h, gidx):  # z_base at global J index: local, else a neighbour's edge
            if a <= gidx < b:
                return z[h, gidx - a]
            for s in range(world):
                so, sn = int(E[s, h, 2 * R]), int(E[s, h, 2 * R + 1])
                if so <= gidx < so + sn:
                    li = gidx - so
                    return E[s, h, li] if li < R else E[s, h, R + li - (sn - R)]
            raise AssertionError(gidx)

        zn = np.empty_like(z)
        for h in range(H):
            for j in range(n):
                gj = a + j
                m = max(zg(h, i) for i in range(max(0, gj - R), min(ng - 1, gj + R) + 1))
                zn[h, j] = z[h, j] - 0.5 * (m - z[h, j])
        mxh = zn.max(0)
        e = np.exp(zn - mxh)
        zadj = zn + 0.35 * np.log(np.maximum(e / e.sum(0), eps))
        # local top-k candidates (score desc, position asc), padded, all-gather
        cs = np.full((H, K), -np.inf)
        cp = np.zeros((H, K), np.int32)
        for h in range(H):
            order = sorted(range(n), key=lambda j: (-zadj[h, j], j))[:K]
            order.sort()
            cs[h, : len(order)] = zadj[h, order]
            cp[h, : len(order)] = allowed[a + np.array(order, dtype=int)] if order else []
        cs_all = torch.zeros(world, H, K, dtype=torch.float64)
        cp_all = torch.zeros(world, H, K, dtype=torch.int32)
        all_gather_blocks(torch.from_numpy(cs), cs_all)
        all_gather_blocks(torch.from_numpy(cp), cp_all)
        # pick: global top-K of the rank-ordered candidates, keep own positions
        ref, _ = O.load("best").run_selector(vals, allowed, norms, O.make_cfg(k_budget=K))
        ok = True
        for h in range(H):
            sc = cs_all[:, h].reshape(-1).numpy()
            ps = cp_all[:, h].reshape(-1).numpy()
            idx = sorted(range(len(sc)), key=lambda i: (-sc[i], i))[:K]
            mine = sorted(ps[i] for i in idx if ps[i] != 0 and allowed[a] <= ps[i] <= (allowed[b - 1] if n else -1))
            want = [p_ for p_ in ref[h] if (n and allowed[a] <= p_ <= allowed[b - 1])]
            ok &= list(mine) == list(want)
        q.put((rank, bool(ok)))
        dist.destroy_process_group()
    except Exception:  # pragma: no cover
        import traceback

        q.put((rank, traceback.format_exc()))


@pytest.mark.parametrize("cuts", [[0, 1300, 2500], [0, 900, 901, 2500]])
def test_sequence_sharded_selector_protocol_gloo(cuts):
    world = len(cuts) - 1
    ctx = mp.get_context("spawn")
    qu = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_seq_protocol_worker, args=(r, world, port, cuts, qu)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(qu.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {r: True for r in range(world)}, res

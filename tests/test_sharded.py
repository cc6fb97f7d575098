"""Multi-GPU paths — KV-head sharding (C3).

CPU (gloo, world size 2): the exchange protocol of the head-sharded Selector
with the oracle as the per-shard compute (z_base of own heads -> all-gather in
rank order -> soft-NMS + cross-head over all heads -> own top-k) equals the
unsharded reference Selector.
GPU: the device kernels through sfi_selector_fuse / sfi_selector_finish are
bit-identical to the unsharded sfi_selector (P simulated shards in one process,
and two real processes sharing cuda:0 over gloo).
"""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from helpers import oracle


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _init(rank, world, port, backend="gloo"):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group(backend, rank=rank, world_size=world)


def test_head_range():
    from paper_2603_12038_b200.sharded import head_range

    assert [head_range(8, 4, r) for r in range(4)] == [(0, 2), (2, 4), (4, 6), (6, 8)]
    assert head_range(8, 1, 0) == (0, 8)
    with pytest.raises(ValueError):
        head_range(8, 3, 0)


def _case(seed=3, H=8, n=3000):
    rng = np.random.default_rng(seed)
    vals = rng.normal(0.0, 0.4, size=(H, n))
    norms = np.abs(rng.normal(11.0, 2.0, size=(H, n))) + 0.1
    allowed = np.arange(5, 5 + n, dtype=np.int32)
    return vals, norms, allowed


def _protocol_worker(rank, world, port, q):
    try:
        _init(rank, world, port)
        from oracle import oracle as O
        from paper_2603_12038_b200.sharded import all_gather_blocks, head_range

        orc = O.load("best")
        vals, norms, allowed = _case()
        H, n = vals.shape
        cfg = O.make_cfg(k_budget=200)
        h0, h1 = head_range(H, world, rank)
        _, st = orc.run_selector(vals[h0:h1], allowed, norms[h0:h1], cfg, stages=True)
        z_local = torch.from_numpy(st["z_base"]).reshape(1, h1 - h0, n)  # [B=1][H/P][n]
        z_all = torch.empty((world, 1, h1 - h0, n), dtype=torch.float64)
        all_gather_blocks(z_local, z_all)
        z = z_all.permute(1, 0, 2, 3).reshape(H, n).numpy()   # global head order
        z_nms = np.stack([orc.refine_soft_nms(z[h], cfg) for h in range(H)])
        z_adj = orc.refine_cross_head(z_nms, cfg)
        mine = [orc.select_top_k(z_adj[h], allowed, cfg.k_budget) for h in range(h0, h1)]
        full, _ = orc.run_selector(vals, allowed, norms, cfg)
        q.put((rank, all(np.array_equal(a, b) for a, b in zip(mine, full[h0:h1]))))
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, repr(e)))


def test_head_sharded_selector_protocol_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_protocol_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {0: True, 1: True}, res


# ---------------------------------------------------------------- GPU ----

def _full_selector_case(B=2, H=8, Hq=16, lens=(6000, 4100), K=256, Lmax=6200):
    from paper_2603_12038_b200 import SelectorParams, SfiCache

    c = SfiCache(1, B, H, Hq, 128, Lmax, 4, K, 64)
    c.fill_synthetic(seed=11, length=max(lens))
    c.set_lengths(list(lens), [4] * B)
    q = torch.randn(B, Hq, 128, generator=torch.Generator().manual_seed(2)).cuda()
    out = torch.zeros_like(q)
    logits = torch.zeros_like(c.pooled_logits)
    c.dense_decode(0, q, out, logits, 0)
    c.selector(0, logits, SelectorParams())
    torch.cuda.synchronize()
    c.check_errors()
    return c, logits


@pytest.mark.gpu
@pytest.mark.parametrize("P", [2, 4, 8])
def test_head_sharded_selector_bit_exact_simulated(P):
    from paper_2603_12038_b200 import SelectorParams, SfiCache

    B, H, Hq, lens, K, Lmax = 2, 8, 16, (6000, 4100), 256, 6200
    full, logits = _full_selector_case(B, H, Hq, lens, K, Lmax)
    Hl = H // P
    shards, zs = [], []
    for s in range(P):
        c = SfiCache(1, B, Hl, Hl * Hq // H, 128, Lmax, 4, K, 64)
        c.key_norms.copy_(full.key_norms[:, :, s * Hl:(s + 1) * Hl])
        c.set_lengths(list(lens), [4] * B)
        z = c.selector_fuse(0, logits[:, s * Hl:(s + 1) * Hl].contiguous(), SelectorParams())
        zs.append(z.clone())
        shards.append(c)
    z_all = torch.stack(zs)  # [P][B][Hl][Lmax], what the all-gather produces
    for s, c in enumerate(shards):
        c.selector_finish(0, z_all, P, s, SelectorParams())
        torch.cuda.synchronize()
        c.check_errors()
        for b in range(B):
            for hl in range(Hl):
                h = s * Hl + hl
                n_full, n_sh = int(full.n_sel[0, b, h]), int(c.n_sel[0, b, hl])
                assert n_full == n_sh
                assert torch.equal(full.sel[0, b, h, :n_full].cpu(), c.sel[0, b, hl, :n_sh].cpu()), (s, b, hl)


def _gpu_worker(rank, world, port, q, peer=False):
    try:
        _init(rank, world, port)
        torch.cuda.set_device(0)
        from paper_2603_12038_b200 import SelectorParams
        from paper_2603_12038_b200.sharded import HeadShardedSfi

        B, H, Hq, L0, K, Lmax, d = 2, 4, 8, 3000, 128, 3200, 128
        sh = HeadShardedSfi(2, B, H, Hq, d, Lmax, 4, K, 64, peer=peer)
        g = torch.Generator().manual_seed(99)  # identical full data on every rank
        kf = torch.randn(B, H, L0, d, generator=g).bfloat16()
        vf = torch.randn(B, H, L0, d, generator=g).bfloat16()
        qf = torch.randn(B, Hq, d, generator=g)
        norms = kf.double().pow(2).sum(-1).sqrt()  # k^2 exact in fp64; order-free is fine for a Selector input
        for layer in range(2):  # the same data in both layers: peer mode uses one z_base slot per layer
            sh.k_cache[layer, :, :, :L0] = kf[:, sh.h0:sh.h1].cuda()
            sh.v_cache[layer, :, :, :L0] = vf[:, sh.h0:sh.h1].cuda()
            sh.key_norms[layer, :, :, :L0] = norms[:, sh.h0:sh.h1].cuda()
        sh.set_lengths([L0] * B, [4] * B)
        out = torch.zeros(B, sh.local_heads * sh.G, d, device="cuda")
        logits = torch.zeros_like(sh.pooled_logits)
        for layer in (0, 1, 0, 1):
            sh.dense_decode(layer, qf[:, sh.q_slice()].contiguous().cuda(), out, logits, 0)
            sh.selector(layer, logits, SelectorParams())
        torch.cuda.synchronize()
        sh.check_errors()
        same_layers = torch.equal(sh.sel[0], sh.sel[1]) and torch.equal(sh.n_sel[0], sh.n_sel[1])
        # rank 0 checks every shard's indices against the reference on the gathered logits
        nJ = L0 - 64 - 4
        lg = [torch.zeros(B, H // world, Lmax) for _ in range(world)]
        dist.all_gather(lg, logits.cpu())
        sel = [torch.zeros(B, H // world, K, dtype=torch.int32) for _ in range(world)]
        dist.all_gather(sel, sh.sel[0].cpu())
        cnt = [torch.zeros(B, H // world, dtype=torch.int32) for _ in range(world)]
        dist.all_gather(cnt, sh.n_sel[0].cpu())
        ok = True
        if rank == 0:
            from oracle import oracle as O

            orc = O.load("best")
            lg_all = torch.cat(lg, 1)
            sel_all, cnt_all = torch.cat(sel, 1), torch.cat(cnt, 1)
            for b in range(B):
                want, _ = orc.run_selector(lg_all[b, :, :nJ].double().numpy(), np.arange(5, 5 + nJ),
                                           norms[b, :, 4:4 + nJ].numpy(), O.make_cfg(k_budget=K))
                for h in range(H):
                    ok &= np.array_equal(sel_all[b, h, : int(cnt_all[b, h])].numpy(), want[h])
        q.put((rank, bool(ok and same_layers)))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover
        import traceback

        q.put((rank, traceback.format_exc()))


@pytest.mark.gpu
@pytest.mark.parametrize("peer", [False, True])
def test_head_sharded_two_processes_one_gpu(peer):
    """z_base exchanged by all-gather, or in place over CUDA-IPC-mapped peer memory."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gpu_worker, args=(r, 2, port, q, peer)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {0: True, 1: True}, res


# ---- peer-memory setup: ranks fall back together (no split decision) ----

def _agree_worker(rank, world, port, fail_rank, q):
    try:
        _init(rank, world, port)
        from paper_2603_12038_b200.sharded import agree

        raised = False
        try:
            agree(rank != fail_rank, None, "probe", "injected" if rank == fail_rank else "")
        except RuntimeError:
            raised = True
        # both ranks continue with the same collective sequence afterwards (no hang)
        t = torch.tensor([rank], dtype=torch.int32)
        dist.all_reduce(t)
        q.put((rank, (raised, int(t.item()))))
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover
        q.put((rank, repr(e)))


@pytest.mark.parametrize("fail_rank", [-1, 0, 1])
def test_peer_setup_vote_gloo_world2(fail_rank):
    """sharded.agree: a step of the peer-memory setup that fails on ONE rank makes
    every rank raise (and fall back to the all-gather path), never just that one
    (a one-sided fallback left the other rank blocked in a collective)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_agree_worker, args=(r, 2, port, fail_rank, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    want = (fail_rank >= 0, 1)
    assert res == {0: want, 1: want}, res

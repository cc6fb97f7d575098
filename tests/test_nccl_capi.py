"""The C ABI's NCCL entry points (sfi_selector_sharded_nccl, sfi_merge_partials_nccl,
sfi_seq_selector_nccl) on a real NCCL communicator — torch's ProcessGroupNCCL
communicator handed over as an ncclComm_t — at world size 1 (gpurun has one GPU;
NCCL refuses two ranks on one device). The exchange is then a copy, so the
sharded drivers must reproduce the unsharded device path bit for bit; this pins
the NCCL plumbing (run-time symbol resolution, the communicator pointer, the
in-call ncclAllGather on the compute stream) that the multi-GPU runs use.
"""
from __future__ import annotations

import os
import socket

import pytest

pytestmark = pytest.mark.gpu


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(port, res_q):
    try:
        import torch
        import torch.distributed as dist

        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        torch.cuda.set_device(0)
        dist.init_process_group("nccl", rank=0, world_size=1)
        from paper_2603_12038_b200 import SelectorParams, SfiCache
        from paper_2603_12038_b200.sharded import HeadShardedSfi, SeqShardedSfi

        L, B, H, Hq, d, ctx, ns, K, R = 2, 2, 4, 16, 128, 5000, 4, 256, 64
        lens = [ctx, ctx - 900]
        g = torch.Generator().manual_seed(3)
        q = torch.randn(B, Hq, d, generator=g).cuda()
        kn = torch.randn(B, H, d, generator=g).bfloat16().cuda()
        prm = SelectorParams()

        def run(c, drv):
            c.fill_synthetic(seed=11, length=ctx)
            drv.set_lengths(lens, [ns] * B)
            drv.step_advance()
            out = torch.zeros(B, Hq, d, device="cuda")
            lg = torch.zeros_like(c.pooled_logits)
            for l in range(L):
                drv.ring_append(l, kn, kn)
                drv.dense_decode(l, q, out, lg, 0)
                drv.selector(l, lg, prm)
            torch.cuda.synchronize()
            c.check_errors()
            return out.clone(), c.sel.clone(), c.n_sel.clone()

        ref = SfiCache(L, B, H, Hq, d, ctx + 8, ns, K, R)
        o_ref, s_ref, n_ref = run(ref, ref)
        hs = HeadShardedSfi(L, B, H, Hq, d, ctx + 8, ns, K, R, nccl=True)
        assert hs.comm != 0
        o_h, s_h, n_h = run(hs.cache, hs)
        ok_heads = torch.equal(s_h, s_ref) and torch.equal(n_h, n_ref) and torch.equal(o_h, o_ref)
        ss = SeqShardedSfi(L, B, H, Hq, d, ctx + 8, ctx, ns, K, R, nccl=True)
        o_s, s_s, n_s = run(ss.cache, ss)
        ok_seq = torch.equal(s_s, s_ref) and torch.equal(n_s, n_ref)
        err_seq = float((o_s - o_ref).abs().max() / o_ref.abs().max())
        dist.destroy_process_group()
        res_q.put(("ok", ok_heads, ok_seq, err_seq))
    except Exception as e:  # pragma: no cover - reported to the parent
        import traceback

        res_q.put(("error", repr(e), traceback.format_exc()))


def test_nccl_capi_world1_matches_unsharded():
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_worker, args=(_free_port(), q))
    p.start()
    res = q.get(timeout=240)
    p.join(timeout=60)
    assert res[0] == "ok", res
    _, ok_heads, ok_seq, err_seq = res
    assert ok_heads, "KV-head sharded Selector over NCCL != unsharded"
    assert ok_seq, "sequence-sharded Selector over NCCL != unsharded"
    assert err_seq < 1e-5, err_seq

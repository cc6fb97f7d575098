"""The sharded classes themselves over gloo, world size 2 (CPU).

`HeadShardedSfi.selector` and `SeqShardedSfi.selector` (sharded.py) are driven
as they are — their own exchange sequence through `all_gather_blocks` on the
real gloo collectives — with the per-shard device kernels replaced by CPU
stand-ins computed from the oracle (tests only; the product classes have no
CPU path):

* head sharding (C3): the shard's cache is a stand-in whose `selector_fuse`
  returns the reference Selector's z_base for the shard's own heads and whose
  `selector_finish` runs soft-NMS + cross-head over the gathered heads and the
  top-k of its own heads; the selected indices equal the unsharded reference
  run_selector (`proj/src/selector.cpp:204-230`, the cross-head coupling);
* sequence sharding (C4): the three phase methods (`sel_stats` phase 1 / 3,
  `sel_finish`, `sel_pick`) are restated on the shard's slice of J in numpy
  (selector.cu's decode fast path); `selector` itself runs the row-statistics,
  edges and candidate all-gathers in its order, and each shard keeps exactly
  the reference's indices that fall inside it.
"""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _case(seed, H, n):
    rng = np.random.default_rng(seed)
    vals = rng.normal(0.0, 0.4, size=(H, n))
    norms = np.abs(rng.normal(11.0, 2.0, size=(H, n))) + 0.1
    return vals, norms, np.arange(5, 5 + n, dtype=np.int32)


def _run(worker, world, *args):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=worker, args=(r, world, port, q) + args) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {r: True for r in range(world)}, res


def _init(rank, world, port):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)


# ---------------------------------------------------------------- heads ----

class _HeadShardCache:
    """CPU stand-in for the shard's SfiCache: the two calls HeadShardedSfi.selector
    makes, computed by the oracle on the shard's heads."""

    def __init__(self, orc, cfg, vals, norms, allowed, h0, h1):
        self.orc, self.cfg = orc, cfg
        self.vals, self.norms, self.allowed = vals, norms, allowed
        self.h0, self.h1 = h0, h1
        self.sel = None

    def selector_fuse(self, layer, logits, params):
        _, st = self.orc.run_selector(self.vals[self.h0:self.h1], self.allowed, self.norms[self.h0:self.h1],
                                      self.cfg, stages=True)
        n = self.vals.shape[1]
        return torch.from_numpy(st["z_base"]).reshape(1, self.h1 - self.h0, n)  # [B = 1][H / P][n]

    def selector_finish(self, layer, z_all, world, rank, params):
        H = self.vals.shape[0]
        z = z_all.permute(1, 0, 2, 3).reshape(H, -1).numpy()  # rank order = global head order
        z_nms = np.stack([self.orc.refine_soft_nms(z[h], self.cfg) for h in range(H)])
        z_adj = self.orc.refine_cross_head(z_nms, self.cfg)
        self.sel = [self.orc.select_top_k(z_adj[h], self.allowed, self.cfg.k_budget) for h in range(self.h0, self.h1)]


def _head_worker(rank, world, port, q):
    try:
        _init(rank, world, port)
        from oracle import oracle as O
        from paper_2603_12038_b200.sharded import HeadShardedSfi, head_range

        orc = O.load("best")
        vals, norms, allowed = _case(3, 8, 3000)
        H, n = vals.shape
        cfg = O.make_cfg(k_budget=200)
        sh = HeadShardedSfi.__new__(HeadShardedSfi)  # the class's selector, a CPU cache under it
        sh.group, sh.world, sh.rank = None, world, rank
        sh.h0, sh.h1 = head_range(H, world, rank)
        sh.comm, sh.px = 0, None
        sh.cache = _HeadShardCache(orc, cfg, vals, norms, allowed, sh.h0, sh.h1)
        sh.z_all = torch.empty((world, 1, sh.h1 - sh.h0, n), dtype=torch.float64)
        sh.selector(0, None, None)
        full, _ = orc.run_selector(vals, allowed, norms, cfg)
        q.put((rank, all(np.array_equal(a, b) for a, b in zip(sh.cache.sel, full[sh.h0:sh.h1]))))
        dist.destroy_process_group()
    except Exception:  # pragma: no cover - reported to the parent
        import traceback

        q.put((rank, traceback.format_exc()))


def test_head_sharded_class_selector_gloo_world2():
    _run(_head_worker, 2)


# ------------------------------------------------------------- sequence ----

K_SEQ, R_NMS, EPS = 300, 2, 1e-8


def _seq_shard_class():
    from paper_2603_12038_b200.sharded import SeqShardedSfi

    class CpuSeqShard(SeqShardedSfi):
        """SeqShardedSfi with its three per-shard phases restated in numpy on the
        shard's slice [a, b) of J (B = 1); `selector` and its exchanges are the
        class's own."""

        def __init__(self, vals, norms, allowed, a, b, world, rank):
            self.group, self.world, self.rank, self.comm, self.px = None, world, rank, 0, None
            self.vals, self.norms, self.allowed, self.a, self.b = vals, norms, allowed, a, b
            H = vals.shape[0]
            f64 = torch.float64
            self.row_stats, self.stats_all = torch.zeros(H * 6, dtype=f64), torch.zeros(world, H * 6, dtype=f64)
            ne = H * (2 * R_NMS + 2)
            self.edges, self.edges_all = torch.zeros(ne, dtype=f64), torch.zeros(world, ne, dtype=f64)
            self.cand_score, self.cand_pos = torch.zeros(H * K_SEQ, dtype=f64), torch.zeros(H * K_SEQ, dtype=torch.int32)
            self.cand_score_all = torch.zeros(world, H * K_SEQ, dtype=f64)
            self.cand_pos_all = torch.zeros(world, H * K_SEQ, dtype=torch.int32)
            self.picked = None

        def sel_stats(self, layer, logits, phase, params=None):
            H, ng = self.vals.shape
            a, b = self.a, self.b
            v, nm, n = self.vals[:, a:b], self.norms[:, a:b], b - a
            u = (np.arange(a, b) / ((ng - 1) + EPS))[None, :]
            w = (1.0 / (nm + EPS)) * np.exp(-(u * u)) * np.sqrt(1.0 - u + EPS)
            if phase == 1:  # local max + the five sums relative to it
                ml = np.maximum(v.max(1) if n else -1e30, -1e30).astype(np.float64)
                pl = np.exp(v - ml[:, None])
                st = np.stack([ml, pl.sum(1), w.sum(1), (pl * pl).sum(1), (pl * w).sum(1), (w * w).sum(1)], 1)
                self.row_stats.copy_(torch.from_numpy(st.reshape(-1)))
                return
            SA = self.stats_all.numpy().reshape(self.world, H, 6)  # combined in rank order at the global max
            M = SA[:, :, 0].max(0)
            e = np.exp(SA[:, :, 0] - M[None, :])
            S = np.stack([(SA[:, :, 1] * e).sum(0), SA[:, :, 2].sum(0), (SA[:, :, 3] * e * e).sum(0),
                          (SA[:, :, 4] * e).sum(0), SA[:, :, 5].sum(0)], 1)
            p = np.exp(v - M[:, None])
            c1, c2 = 1.0 / S[:, 0], 1.0 / S[:, 1]
            ff, fr, rr = S[:, 2] * c1 * c1, S[:, 3] * c1 * c2, S[:, 4] * c2 * c2
            den = ff - 2 * fr + rr
            lam = np.where(np.abs(den) >= EPS, np.clip((ff - fr) / np.where(den == 0, 1, den), 0, 0.02), 0.0)
            self.z = np.log((1 - lam)[:, None] * c1[:, None] * p + lam[:, None] * c2[:, None] * w + EPS)
            edge = np.full((H, 2 * R_NMS + 2), np.nan)  # first R, last R, offset, count
            for h in range(H):
                for t in range(R_NMS):
                    if t < n:
                        edge[h, t] = self.z[h, t]
                    if 0 <= n - R_NMS + t < n:
                        edge[h, R_NMS + t] = self.z[h, n - R_NMS + t]
                edge[h, 2 * R_NMS], edge[h, 2 * R_NMS + 1] = a, n
            self.edges.copy_(torch.from_numpy(edge.reshape(-1)))

        def sel_finish(self, layer, params=None):
            H, ng = self.vals.shape
            a, b, z = self.a, self.b, self.z
            n = b - a
            E = self.edges_all.numpy().reshape(self.world, H, 2 * R_NMS + 2)

            def zg(h, gidx):  # z_base at a global J index: own slice, else a neighbour's edge
                if a <= gidx < b:
                    return z[h, gidx - a]
                for s in range(self.world):
                    so, sn = int(E[s, h, 2 * R_NMS]), int(E[s, h, 2 * R_NMS + 1])
                    if so <= gidx < so + sn:
                        li = gidx - so
                        return E[s, h, li] if li < R_NMS else E[s, h, R_NMS + li - (sn - R_NMS)]
                raise AssertionError(gidx)

            zn = np.empty_like(z)
            for h in range(H):
                for j in range(n):
                    gj = a + j
                    m = max(zg(h, i) for i in range(max(0, gj - R_NMS), min(ng - 1, gj + R_NMS) + 1))
                    zn[h, j] = z[h, j] - 0.5 * (m - z[h, j])
            e = np.exp(zn - zn.max(0))
            zadj = zn + 0.35 * np.log(np.maximum(e / e.sum(0), EPS))
            cs = np.full((H, K_SEQ), -np.inf)
            cp = np.zeros((H, K_SEQ), np.int32)
            for h in range(H):
                order = sorted(sorted(range(n), key=lambda j: (-zadj[h, j], j))[:K_SEQ])
                cs[h, :len(order)] = zadj[h, order]
                cp[h, :len(order)] = self.allowed[a + np.array(order, dtype=int)] if order else []
            self.cand_score.copy_(torch.from_numpy(cs.reshape(-1)))
            self.cand_pos.copy_(torch.from_numpy(cp.reshape(-1)))

        def sel_pick(self, layer):
            H = self.vals.shape[0]
            cs = self.cand_score_all.numpy().reshape(self.world, H, K_SEQ)
            cp = self.cand_pos_all.numpy().reshape(self.world, H, K_SEQ)
            lo, hi = (self.allowed[self.a], self.allowed[self.b - 1]) if self.b > self.a else (1, 0)
            self.picked = []
            for h in range(H):
                sc, ps = cs[:, h].reshape(-1), cp[:, h].reshape(-1)
                idx = sorted(range(len(sc)), key=lambda i: (-sc[i], i))[:K_SEQ]
                self.picked.append(sorted(int(ps[i]) for i in idx if ps[i] != 0 and lo <= ps[i] <= hi))

    return CpuSeqShard


def _seq_worker(rank, world, port, q, cuts):
    try:
        _init(rank, world, port)
        from oracle import oracle as O

        vals, norms, allowed = _case(4, 4, 2500)
        sh = _seq_shard_class()(vals, norms, allowed, cuts[rank], cuts[rank + 1], world, rank)
        sh.selector(0, None, None)
        ref, _ = O.load("best").run_selector(vals, allowed, norms, O.make_cfg(k_budget=K_SEQ))
        lo_i, hi_i = cuts[rank], cuts[rank + 1]
        ok = True
        for h in range(vals.shape[0]):
            want = [int(p) for p in ref[h] if hi_i > lo_i and allowed[lo_i] <= p <= allowed[hi_i - 1]]
            ok &= sh.picked[h] == want
        q.put((rank, bool(ok)))
        dist.destroy_process_group()
    except Exception:  # pragma: no cover
        import traceback

        q.put((rank, traceback.format_exc()))


@pytest.mark.parametrize("cuts", [[0, 1300, 2500], [0, 900, 901, 2500]])
def test_seq_sharded_class_selector_gloo(cuts):
    _run(_seq_worker, len(cuts) - 1, cuts)

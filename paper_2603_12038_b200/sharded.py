"""Multi-GPU SFI decode: one process per GPU, torch.distributed for
the plumbing (NCCL over NVLink on B200 boxes; gloo for CPU-side tests).

KV-head sharding (config C3): rank r of P holds KV heads [r*H/P, (r+1)*H/P) of
every layer and request (and their G query heads each). Attention, key norms,
the ring, the compact builder and every Selector stage except cross-head
exclusivity are per head, so fast steps exchange nothing. Cross-head
exclusivity (selector.cpp:204-230) is a softmax over all KV heads of a request
at each position: per layer and slow step the ranks all-gather the Selector's
z_base blocks (fp64 [B][H/P][max_positions]) and each finishes soft-NMS +
cross-head in global head order and the top-k of its own heads — indices
bit-identical to the 1-GPU Selector.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

from .device import SfiCache


def head_range(n_kv_heads: int, world: int, rank: int) -> tuple[int, int]:
    """KV heads owned by `rank` (contiguous, equal blocks)."""
    if n_kv_heads % world != 0:
        raise ValueError(f"{n_kv_heads} KV heads do not split over {world} ranks")
    per = n_kv_heads // world
    return rank * per, (rank + 1) * per


def all_gather_blocks(local: torch.Tensor, out: torch.Tensor, group=None) -> torch.Tensor:
    """out[r] = local of rank r (rank order). NCCL gathers in place on the current
    stream; gloo (CPU tests) stages CUDA tensors through host memory."""
    backend = dist.get_backend(group)
    if backend == "nccl" or not local.is_cuda:
        dist.all_gather_into_tensor(out.view(-1), local.contiguous().view(-1), group=group)
        return out
    host = torch.empty_like(out, device="cpu")
    dist.all_gather_into_tensor(host.view(-1), local.detach().cpu().contiguous().view(-1), group=group)
    out.copy_(host)
    return out


def nccl_comm_ptr(group=None) -> int:
    """The ncclComm_t of torch's NCCL process group (as an integer), for the C
    ABI's NCCL entry points (sfi_selector_sharded_nccl, sfi_merge_partials_nccl,
    sfi_seq_selector_nccl). torch creates communicators lazily: one tiny
    collective first makes sure this one exists."""
    pg = group if group is not None else dist.distributed_c10d._get_default_group()
    if dist.get_backend(group) != "nccl":
        raise RuntimeError("the C-ABI NCCL exchange needs the nccl backend")
    t = torch.zeros(1, device=torch.device("cuda", torch.cuda.current_device()))
    dist.all_reduce(t, group=group)
    torch.cuda.synchronize()
    ptr = pg._get_backend(torch.device("cuda"))._comm_ptr()
    if not ptr:
        raise RuntimeError("ProcessGroupNCCL has no communicator for this device")
    return int(ptr)


def agree(ok: bool, group=None, what: str = "peer-memory setup", err: str = "") -> None:
    """Every rank votes (all_reduce MIN); raises on EVERY rank unless all succeeded,
    so ranks fall back to the all-gather path together instead of some blocking
    in a collective the others never enter."""
    dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(group) == "nccl" \
        else torch.device("cpu")
    t = torch.tensor([1 if ok else 0], dtype=torch.int32, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MIN, group=group)
    if int(t.item()) != 1:
        raise RuntimeError(f"{what} failed on at least one rank" + (f" (here: {err})" if err else ""))


def _attempt(fn):
    try:
        return True, "", fn()
    except Exception as e:  # noqa: BLE001 - reported through the vote
        return False, f"{type(e).__name__}: {e}", None


def _enable_peer_access(world: int) -> None:
    """Maps every visible GPU into this process's device (NVLink P2P), so IPC
    buffers opened in another device's context are addressable from kernels on
    ours. One process per GPU: a no-op on a single device."""
    n = min(world, torch.cuda.device_count())
    if n < 2:
        return
    me = torch.cuda.current_device()
    if not all(torch.cuda.can_device_access_peer(me, o) for o in range(n) if o != me):
        raise RuntimeError("peer access between the visible GPUs is not available")
    try:
        from cuda.bindings import runtime as rt
    except ImportError:  # pragma: no cover - cuda-python ships in the image
        from cuda import cudart as rt
    for other in range(n):
        if other != me and torch.cuda.can_device_access_peer(me, other):
            rt.cudaDeviceEnablePeerAccess(other, 0)  # "already enabled" is fine


class PeerExchange:
    """Shard exchanges over peer memory (no collective launch).

    Each rank owns `slots` attention-partial buffers (o fp32 [rows][d], lse fp32
    [rows]; slots = 0 when only blocks are gathered), named `shared` blocks and an
    epoch flag, allocated from the CUDA caching allocator and shared with
    every rank once through CUDA IPC handles (torch.multiprocessing reductions,
    exchanged with all_gather_object). Per exchange a rank writes its partial into
    slot s, bumps its flag (sfi_peer_publish) and merges every rank's slot s in
    place (sfi_peer_merge: acquire the peer flags, read over NVLink, rank order).
    `peers` (lockstep tests in one process): the other shards' PeerExchange
    objects, used directly instead of IPC."""

    def __init__(self, world: int, rank: int, slots: int, rows: int, d: int, device, group=None,
                 peers: list | None = None, shared: dict | None = None):
        from . import _sfi_b200 as _C

        if slots == 1:
            raise ValueError("peer exchange needs >= 2 partial slots (one per layer)")
        self._C, self.world, self.rank, self.slots, self.rows, self.d = _C, world, rank, slots, rows, d
        self.o = torch.zeros(max(slots, 1), max(rows, 1), max(d, 1), dtype=torch.float32, device=device)
        self.lse = torch.zeros(max(slots, 1), max(rows, 1), dtype=torch.float32, device=device)
        self.flag = torch.zeros(64, dtype=torch.int32, device=device)  # [0] used; own 256 B line
        self.shared = dict(shared or {})  # further blocks all-gathered in place (gather())
        self.shared["_probe"] = torch.zeros(64, dtype=torch.int32, device=device)
        self._peer_views = None
        if peers is None:  # every step votes: no rank commits to peer memory alone
            self.connect(self._exchange_handles(group))
            self._self_test(group)

    def _self_test(self, group):
        """One published round trip through every mapping; raises (callers fall
        back to the all-gather path) unless every rank reads every block."""
        probe = self.shared["_probe"]
        probe.fill_(1000 + self.rank)
        seen = torch.full((self.world, 64), -1, dtype=torch.int32, device=probe.device)
        st = torch.cuda.current_stream().cuda_stream
        self.publish(st)
        self.gather("_probe", seen, st)
        want = (1000 + torch.arange(self.world, device=probe.device, dtype=torch.int32))[:, None].expand(-1, 64)
        ok = torch.tensor([int(torch.equal(seen, want))], dtype=torch.int32, device=probe.device)
        if dist.get_backend(group) != "nccl":
            ok = ok.cpu()
        dist.all_reduce(ok, op=dist.ReduceOp.MIN, group=group)
        if int(ok.item()) != 1:
            raise RuntimeError("peer-memory self-test failed: a rank could not read every mapped block")

    def _exchange_handles(self, group):
        from torch.multiprocessing.reductions import reduce_tensor

        ok, err, mine = _attempt(lambda: (_enable_peer_access(self.world),
                                          [reduce_tensor(t) for t in self.local_views()])[1])
        agree(ok, group, "P2P access / IPC handle export", err)
        objs = [None] * self.world
        dist.all_gather_object(objs, mine, group=group)

        def open_all():
            return [self.local_views() if r == self.rank else tuple(fn(*args) for fn, args in rec)
                    for r, rec in enumerate(objs)]
        ok, err, views = _attempt(open_all)
        agree(ok, group, "IPC handle import", err)
        return views

    def local_views(self):
        return (self.o, self.lse, self.flag, *self.shared.values())

    def connect(self, views):
        """views[r] = (o, lse, flag) of rank r as addressable from this process."""
        self._peer_views = views  # keeps the IPC mappings alive
        dev = self.o.device
        ptr = lambda xs: torch.tensor(xs, dtype=torch.int64, device=dev)  # noqa: E731
        self.o_ptrs = ptr([[v[0][s].data_ptr() for v in views] for s in range(self.slots)])
        self.lse_ptrs = ptr([[v[1][s].data_ptr() for v in views] for s in range(self.slots)])
        self.flag_ptrs = ptr([v[2].data_ptr() for v in views])
        self.src_ptrs = {name: ptr([v[3 + i].data_ptr() for v in views]) for i, name in enumerate(self.shared)}

    def publish(self, stream: int):
        self._C.peer_publish(self.flag.data_ptr(), stream)

    def gather(self, name: str, dst: torch.Tensor, stream: int):
        """dst[r] = rank r's block `name`, read in place once rank r published."""
        t = self.shared[name]
        self._C.peer_gather(self.world, t.numel() * t.element_size(), self.src_ptrs[name].data_ptr(),
                            self.flag_ptrs.data_ptr(), self.flag.data_ptr(), dst.data_ptr(), stream)

    def merge(self, slot: int, out_ptr: int, stream: int):
        self._C.peer_merge(self.world, self.rows, self.d, self.o_ptrs[slot].data_ptr(),
                           self.lse_ptrs[slot].data_ptr(), self.flag_ptrs.data_ptr(), self.flag.data_ptr(),
                           out_ptr, stream)


def connect_lockstep(shards) -> None:
    """Wires the PeerExchange of P lockstep shards of one process to each other."""
    views = [s.px.local_views() for s in shards]
    for s in shards:
        s.px.connect(views)


class HeadShardedSfi:
    """This rank's shard of a KV-head-sharded SFI cache (n_layers x batch x
    n_kv_heads/P heads). Same step API as SfiCache; only the Selector talks to
    the other ranks."""

    def __init__(self, n_layers: int, batch: int, n_kv_heads: int, n_q_heads: int, head_dim: int,
                 max_positions: int, n_sink: int = 4, k_budget: int = 2048, n_recent: int = 256,
                 group=None, device=None, peer: bool = False, nccl: bool = False):
        """peer=True: the Selector's z_base all-gather reads every rank's block in
        place over peer memory (PeerExchange: CUDA IPC, sfi_peer_gather), one
        block slot per layer so a block is only rewritten after every rank read it.
        nccl=True: the C ABI's sfi_selector_sharded_nccl does fuse + ncclAllGather
        + finish in one call on torch's NCCL communicator (graph capturable).
        Otherwise torch.distributed all-gathers the blocks."""
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.h0, self.h1 = head_range(n_kv_heads, self.world, self.rank)
        G = n_q_heads // n_kv_heads
        self.n_kv_heads, self.n_q_heads, self.G = n_kv_heads, n_q_heads, G
        self.local_heads = self.h1 - self.h0
        if device is None:
            device = torch.device("cuda", torch.cuda.current_device())
        self.cache = SfiCache(n_layers, batch, self.local_heads, self.local_heads * G, head_dim,
                              max_positions, n_sink, k_budget, n_recent, device=device)
        dev = self.cache.k_cache.device
        self.z_all = torch.empty((self.world, batch, self.local_heads, max_positions), dtype=torch.float64,
                                 device=dev)
        self.px = None
        self.comm = nccl_comm_ptr(group) if nccl else 0
        if peer and self.world > 1:
            if n_layers < 2:
                raise ValueError("peer exchange keeps one z_base slot per layer: needs >= 2 layers")
            self.z_slots = torch.zeros((n_layers, batch, self.local_heads, max_positions), dtype=torch.float64,
                                       device=dev)
            self.px = PeerExchange(self.world, self.rank, 0, 0, 0, dev, group,
                                   shared={f"z{l}": self.z_slots[l] for l in range(n_layers)})

    # q heads of this shard: [h0*G, h1*G) of the model's q heads
    def q_slice(self) -> slice:
        return slice(self.h0 * self.G, self.h1 * self.G)

    def selector(self, layer: int, logits: torch.Tensor, params=None):
        if self.comm:
            c = self.cache
            c._C_sel_nccl(layer, logits, params, self.comm, self.world, self.rank, self.z_all)
            return
        z = self.cache.selector_fuse(layer, logits, params)
        if self.px is not None:
            st = self.cache._stream()
            self.z_slots[layer].copy_(z)
            self.px.publish(st)
            self.px.gather(f"z{layer}", self.z_all, st)
            self.cache.selector_finish(layer, self.z_all, self.world, self.rank, params)
        elif self.world > 1:
            all_gather_blocks(z, self.z_all, self.group)
            self.cache.selector_finish(layer, self.z_all, self.world, self.rank, params)
        else:
            self.cache.selector_finish(layer, z.unsqueeze(0), 1, 0, params)

    def __getattr__(self, name):  # everything else is per head: the local cache
        if name == "cache":
            raise AttributeError(name)
        return getattr(self.cache, name)


# ---------------------------------------------------------------------------
# Sequence sharding (config C4: 256K context, too few KV heads to split)

def seq_block(prompt_len: int, world: int) -> int:
    """Positions per non-last shard: the prompt split evenly; decode tokens
    land on the last shard."""
    return -(-prompt_len // world)


class SeqShardedSfi:
    """This rank's shard of a sequence-sharded SFI cache: positions
    (base, base + block] (the last rank: (base, max_positions]) of every
    request, all KV heads. Per layer, slow steps exchange the Selector's row
    statistics (max, 5 sums), soft-NMS edges and top-k candidates; every step
    exchanges the (O, LSE) attention partials, merged in rank order.
    Slow steps add three exchanges per layer: the Selector's row statistics
    (local max + five sums, rescaled to the global max on arrival), the
    soft-NMS edges and the top-k candidates.

    The collective steps are separate methods so a single process can drive
    P shards in lockstep (tests); `selector`, `dense_decode` and `fast_decode`
    run them with torch.distributed on the current stream."""

    def __init__(self, n_layers: int, batch: int, n_kv_heads: int, n_q_heads: int, head_dim: int,
                 max_positions: int, prompt_len: int, n_sink: int = 4, k_budget: int = 2048,
                 n_recent: int = 256, group=None, device=None, world: int | None = None,
                 rank: int | None = None, peer: bool = False, peers: list | None = None, nccl: bool = False):
        """peer=True: the per-step (O, LSE) exchange goes through PeerExchange
        (peer memory, no collective launch); `peers` wires lockstep shards of
        one process to each other instead of through IPC."""
        from . import _sfi_b200 as _C

        self._C = _C
        self.group = group
        self.world = world if world is not None else dist.get_world_size(group)
        self.rank = rank if rank is not None else dist.get_rank(group)
        self.block = seq_block(prompt_len, self.world)
        self.base = self.rank * self.block
        self.is_last = self.rank == self.world - 1
        cap = (max_positions - self.base) if self.is_last else self.block
        if cap < 1 or (self.is_last and self.base >= prompt_len):
            raise ValueError("sequence shard layout: the prompt must reach the last shard")
        self.cap = cap
        if device is None:
            device = torch.device("cuda", torch.cuda.current_device())
        self.cache = SfiCache(n_layers, batch, n_kv_heads, n_q_heads, head_dim, cap, n_sink, k_budget,
                              n_recent, device=device)
        dev = self.cache.k_cache.device
        B, H, Hq, P, K = batch, n_kv_heads, n_q_heads, self.world, k_budget
        z = lambda *s, dt=torch.int32: torch.zeros(s, dtype=dt, device=dev)  # noqa: E731
        self.g_prefix, self.g_nsink, self.g_recent = z(B), z(B), z(B)
        self.j_off, self.n_glob = z(B), z(B)
        self.params = _C.SelectorParams()
        ne = _C.seq_edges_doubles(self.cache.shape, self.params)
        f64 = torch.float64
        self.row_stats = z(B * H * 6, dt=f64)
        self.stats_all = z(P, B * H * 6, dt=f64)
        self.edges = z(ne, dt=f64)
        self.edges_all = z(P, ne, dt=f64)
        self.cand_score, self.cand_pos = z(B * H * K, dt=f64), z(B * H * K)
        self.cand_score_all, self.cand_pos_all = z(P, B * H * K, dt=f64), z(P, B * H * K)
        self.pick_scratch = z(_C.seq_pick_scratch_bytes(self.cache.shape, P), dt=torch.uint8)
        self.o_part = z(B, Hq, head_dim, dt=torch.float32)
        self.lse_part = z(B, Hq, dt=torch.float32)
        self.o_all = z(P, B, Hq, head_dim, dt=torch.float32)
        self.lse_all = z(P, B, Hq, dt=torch.float32)
        self.n_recent = n_recent
        # nccl=True: every exchange in-call through the C ABI on torch's NCCL communicator
        self.comm = nccl_comm_ptr(group) if nccl else 0
        if self.comm:
            nb = _C.seq_selector_nccl_scratch_bytes(self.cache.shape, self.params, P)
            self.nccl_scratch = z(nb, dt=torch.uint8)
        self.px = None
        if peer or peers is not None:
            if n_layers < 2:  # a slot may only be rewritten once every rank merged it
                raise ValueError("peer exchange keeps one partial slot per layer: needs >= 2 layers")
            self.px = PeerExchange(P, self.rank, max(2, n_layers), B * Hq, head_dim, dev, group,
                                   peers=[] if peers is not None else None,
                                   shared=dict(row_stats=self.row_stats, edges=self.edges,
                                               cand_score=self.cand_score, cand_pos=self.cand_pos))

    # -- lengths -------------------------------------------------------------
    def set_lengths(self, prefix_len, n_sink_b):
        """Global lengths of every request (host values, like SfiCache.set_lengths)."""
        L = torch.tensor(list(map(int, prefix_len)), dtype=torch.int32)
        ns = torch.tensor(list(map(int, n_sink_b)), dtype=torch.int32)
        if self.is_last and int(L.min()) <= self.base:
            raise ValueError("decode appends on the last shard: every prefix must reach it")
        self.g_prefix.copy_(L)
        self.g_nsink.copy_(ns)
        self.g_recent.copy_(torch.clamp(L - ns, 0, self.n_recent))
        self._lengths(0)
        torch.cuda.current_stream().synchronize()

    def _lengths(self, advance: int):
        c = self.cache
        self._C.seq_lengths(c.shape, c.cache, self.g_prefix.data_ptr(), self.g_nsink.data_ptr(),
                            self.g_recent.data_ptr(), advance, self.base, int(self.is_last),
                            self.j_off.data_ptr(), self.n_glob.data_ptr(), c._stream())

    def step_advance(self):
        self._lengths(1)

    # -- attention partials ----------------------------------------------------
    def _part_ptrs(self, layer):
        if self.px is None:
            return self.o_part.data_ptr(), self.lse_part.data_ptr()
        slot = layer % self.px.slots
        return self.px.o[slot].data_ptr(), self.px.lse[slot].data_ptr()

    def dense_partial(self, layer, q, logits, pool=0):
        c = self.cache
        o, lse = self._part_ptrs(layer)
        self._C.dense_decode_partial(c.shape, c.cache, layer, c._ptr(q, torch.float32), o, lse,
                                     c._ptr(logits, torch.float32), pool, c._stream())
        if self.px is not None:
            self.px.publish(c._stream())

    def fast_partial(self, layer, q, k_new, v_new, prefetch=False):
        c = self.cache
        own = self.is_last  # the current position is on the last shard
        o, lse = self._part_ptrs(layer)
        self._C.fast_decode_partial(c.shape, c.cache, layer, c._ptr(q, torch.float32),
                                    c._ptr(k_new, torch.bfloat16) if own else 0,
                                    c._ptr(v_new, torch.bfloat16) if own else 0, o, lse,
                                    self._C.FAST_PREFETCH if prefetch else 0, c._stream())
        if self.px is not None:
            self.px.publish(c._stream())

    def peer_merge(self, layer, out):
        """out = LSE merge of every rank's partial of `layer`, read in place from peer memory."""
        self.px.merge(layer % self.px.slots, self.cache._ptr(out, torch.float32), self.cache._stream())

    def merge(self, out):
        """out = LSE merge of the gathered partials (o_all, lse_all) in rank order."""
        B, Hq, d = self.o_part.shape
        self._C.merge_partials(self.world, B * Hq, d, self.o_all.data_ptr(), self.lse_all.data_ptr(),
                               self.cache._ptr(out, torch.float32), self.cache._stream())

    def _exchange_partials(self):
        all_gather_blocks(self.o_part, self.o_all, self.group)
        all_gather_blocks(self.lse_part, self.lse_all, self.group)

    def _nccl_merge(self, out):
        B, Hq, d = self.o_part.shape
        self._C.merge_partials_nccl(self.world, B * Hq, d, self.o_part.data_ptr(), self.lse_part.data_ptr(),
                                    self.o_all.data_ptr(), self.lse_all.data_ptr(),
                                    self.cache._ptr(out, torch.float32), self.comm, self.cache._stream())

    def dense_decode(self, layer, q, out, logits, pool=0):
        self.dense_partial(layer, q, logits, pool)
        if self.comm:
            self._nccl_merge(out)
            return
        if self.px is not None:
            self.peer_merge(layer, out)
            return
        self._exchange_partials()
        self.merge(out)

    def fast_decode(self, layer, q, k_new, v_new, out, prefetch=False):
        self.fast_partial(layer, q, k_new, v_new, prefetch)
        if self.comm:
            self._nccl_merge(out)
            return
        if self.px is not None:
            self.peer_merge(layer, out)
            return
        self._exchange_partials()
        self.merge(out)

    def ring_append(self, layer, k_new, v_new):
        if self.is_last:
            self.cache.ring_append(layer, k_new, v_new)

    # -- Selector phases ---------------------------------------------------------
    def sel_stats(self, layer, logits, phase, params=None):
        """phase 1: local row statistics (max, five sums relative to it) -> row_stats;
        phase 3: z_base from the all-gathered statistics + soft-NMS edges."""
        c = self.cache
        self._C.seq_selector_stats(c.shape, c.cache, layer, c._ptr(logits, torch.float32),
                                   params or self.params, self.j_off.data_ptr(), self.n_glob.data_ptr(), phase,
                                   self.row_stats.data_ptr(), self.stats_all.data_ptr(), self.world,
                                   self.edges.data_ptr(), c._stream())

    def sel_finish(self, layer, params=None):
        c = self.cache
        self._C.seq_selector_finish(c.shape, c.cache, layer, params or self.params, self.j_off.data_ptr(),
                                    self.n_glob.data_ptr(), self.edges_all.data_ptr(), self.world, self.base,
                                    self.cand_score.data_ptr(), self.cand_pos.data_ptr(), c._stream())

    def sel_pick(self, layer):
        c = self.cache
        self._C.seq_selector_pick(c.shape, c.cache, layer, self.world, self.cand_score_all.data_ptr(),
                                  self.cand_pos_all.data_ptr(), self.base, self.base + self.cap,
                                  self.pick_scratch.data_ptr(), c._stream())

    def selector(self, layer, logits, params=None):
        # three exchanges per layer: row statistics, soft-NMS edges, top-k candidates
        if self.comm:  # all three in one C-ABI call over NCCL
            c = self.cache
            self._C.seq_selector_nccl(c.shape, c.cache, layer, c._ptr(logits, torch.float32), params or self.params,
                                      self.j_off.data_ptr(), self.n_glob.data_ptr(), self.base, self.base + self.cap,
                                      self.comm, self.world, self.nccl_scratch.data_ptr(), self.nccl_scratch.numel(),
                                      c._stream())
            return
        if self.px is not None:  # over peer memory: publish, then gather in place
            st = self.cache._stream()
            self.sel_stats(layer, logits, 1, params)
            self.px.publish(st)
            self.px.gather("row_stats", self.stats_all, st)
            self.sel_stats(layer, logits, 3, params)
            self.px.publish(st)
            self.px.gather("edges", self.edges_all, st)
            self.sel_finish(layer, params)
            self.px.publish(st)
            self.px.gather("cand_score", self.cand_score_all, st)
            self.px.gather("cand_pos", self.cand_pos_all, st)
            self.sel_pick(layer)
            return
        self.sel_stats(layer, logits, 1, params)
        all_gather_blocks(self.row_stats, self.stats_all, self.group)
        self.sel_stats(layer, logits, 3, params)
        all_gather_blocks(self.edges, self.edges_all, self.group)
        self.sel_finish(layer, params)
        all_gather_blocks(self.cand_score, self.cand_score_all, self.group)
        all_gather_blocks(self.cand_pos, self.cand_pos_all, self.group)
        self.sel_pick(layer)

    def __getattr__(self, name):  # compact_build, check_errors, buffers: the local cache
        if name == "cache":
            raise AttributeError(name)
        return getattr(self.cache, name)

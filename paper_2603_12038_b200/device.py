"""Batched device API: one SFI cache (all layers, a batch of requests) whose
buffers are torch tensors in HBM, driven through the C ABI on the current
torch CUDA stream. This is the production / bench path; torch is only the
allocator and the stream provider.

Layout (include/sfi_b200.h):
    k_cache, v_cache  bf16 [L][B][H][max_positions][d]
    key_norms         fp64 [L][B][H][max_positions]
    ck, cv            bf16 [L][B][H][n_recent + n_sink + k_budget][d]
    sel               int32 [L][B][H][k_budget],  n_sel int32 [L][B][H]
    prefix_len, n_sink_b, recent_len  int32 [B]
"""
from __future__ import annotations

import torch

from . import _sfi_b200 as _C


class SfiCache:
    def __init__(self, n_layers: int, batch: int, n_kv_heads: int, n_q_heads: int,
                 head_dim: int, max_positions: int, n_sink: int = 4, k_budget: int = 2048,
                 n_recent: int = 256, device: str | torch.device = "cuda"):
        s = _C.Shape()
        s.n_layers, s.batch, s.n_kv_heads, s.n_q_heads = n_layers, batch, n_kv_heads, n_q_heads
        s.head_dim, s.max_positions = head_dim, max_positions
        s.n_sink, s.k_budget, s.n_recent = n_sink, k_budget, n_recent
        _C.shape_validate(s)
        self.shape = s
        self.sizes = _C.buffer_sizes(s)
        dev = torch.device(device)
        L, B, H, d = n_layers, batch, n_kv_heads, head_dim
        self.compact_rows = n_recent + n_sink + k_budget
        z = torch.zeros
        self.k_cache = z((L, B, H, max_positions, d), dtype=torch.bfloat16, device=dev)
        self.v_cache = z((L, B, H, max_positions, d), dtype=torch.bfloat16, device=dev)
        self.key_norms = z((L, B, H, max_positions), dtype=torch.float64, device=dev)
        self.ck = z((L, B, H, self.compact_rows, d), dtype=torch.bfloat16, device=dev)
        self.cv = z((L, B, H, self.compact_rows, d), dtype=torch.bfloat16, device=dev)
        self.sel = z((L, B, H, max(1, k_budget)), dtype=torch.int32, device=dev)
        self.n_sel = z((L, B, H), dtype=torch.int32, device=dev)
        self.prefix_len = z((B,), dtype=torch.int32, device=dev)
        self.n_sink_b = z((B,), dtype=torch.int32, device=dev)
        self.recent_len = z((B,), dtype=torch.int32, device=dev)
        self.error_flags = z((1,), dtype=torch.int32, device=dev)
        self.workspace = z((self.sizes["workspace"],), dtype=torch.uint8, device=dev)
        self.pooled_logits = z((B, H, max_positions), dtype=torch.float32, device=dev)
        self._bind()

    def _bind(self):
        c = _C.Cache()
        c.k_cache, c.v_cache = self.k_cache.data_ptr(), self.v_cache.data_ptr()
        c.key_norms = self.key_norms.data_ptr()
        c.ck, c.cv = self.ck.data_ptr(), self.cv.data_ptr()
        c.sel, c.n_sel = self.sel.data_ptr(), self.n_sel.data_ptr()
        c.prefix_len, c.n_sink_b = self.prefix_len.data_ptr(), self.n_sink_b.data_ptr()
        c.recent_len = self.recent_len.data_ptr()
        c.error_flags = self.error_flags.data_ptr()
        c.workspace = self.workspace.data_ptr()
        c.workspace_bytes = self.sizes["workspace"]
        self.cache = c

    def layer_batched_view(self) -> "SfiCache":
        """Diagnostic view of all layers as ONE layer of n_layers x batch requests
        (same K/V, compact and selection buffers; own lengths and workspace): one
        launch then streams what a step's per-layer launches stream, which
        measures the kernels without the per-layer launch boundary."""
        s0 = self.shape
        L, B = s0.n_layers, s0.batch
        s = _C.Shape()
        s.n_layers, s.batch, s.n_kv_heads, s.n_q_heads = 1, L * B, s0.n_kv_heads, s0.n_q_heads
        s.head_dim, s.max_positions = s0.head_dim, s0.max_positions
        s.n_sink, s.k_budget, s.n_recent = s0.n_sink, s0.k_budget, s0.n_recent
        _C.shape_validate(s)
        v = SfiCache.__new__(SfiCache)
        v.shape, v.sizes, v.compact_rows = s, _C.buffer_sizes(s), self.compact_rows
        flat = lambda t: t.view(1, L * B, *t.shape[2:])  # noqa: E731
        v.k_cache, v.v_cache, v.key_norms = flat(self.k_cache), flat(self.v_cache), flat(self.key_norms)
        v.ck, v.cv, v.sel, v.n_sel = flat(self.ck), flat(self.cv), flat(self.sel), flat(self.n_sel)
        dev = self.k_cache.device
        v.prefix_len = self.prefix_len.repeat(L)
        v.n_sink_b = self.n_sink_b.repeat(L)
        v.recent_len = self.recent_len.repeat(L)
        v.error_flags = self.error_flags
        v.workspace = torch.zeros((v.sizes["workspace"],), dtype=torch.uint8, device=dev)
        v.pooled_logits = None
        v._bind()
        return v

    # -- plumbing -------------------------------------------------------------
    @staticmethod
    def _stream(stream=None) -> int:
        if stream is None:
            stream = torch.cuda.current_stream()
        return stream.cuda_stream

    @staticmethod
    def _ptr(t: torch.Tensor | None, dtype=None) -> int:
        if t is None:
            return 0
        if not t.is_cuda or not t.is_contiguous():
            raise ValueError("device op arguments must be contiguous CUDA tensors")
        if dtype is not None and t.dtype != dtype:
            raise TypeError(f"expected {dtype}, got {t.dtype}")
        return t.data_ptr()

    # -- C ABI, one to one -----------------------------------------------------
    def set_lengths(self, prefix_len, n_sink_b, recent_len=None, stream=None):
        _C.set_lengths(self.shape, self.cache, list(map(int, prefix_len)), list(map(int, n_sink_b)),
                       None if recent_len is None else list(map(int, recent_len)),
                       self._stream(stream))

    def fill_synthetic(self, seed: int, length: int, stream=None):
        _C.fill_synthetic(self.shape, self.cache, seed, length, self._stream(stream))

    def plant_peaked(self, layer: int, q: torch.Tensor, n_planted: int = 32, scale: float = 3.0,
                     seed: int = 0) -> torch.Tensor:
        """SURVEY §8d "peaked" synthetic inputs: in every (request, KV head) slice,
        n_planted positions drawn from the slice's current J (seeded) get the key
        k = bf16(scale * q_g + N(0, 1)), g cycling over the group's query heads of
        q fp32 [B][Hq][d]; their fp64 key norms are rewritten. Call after
        set_lengths and fill_synthetic. Returns the planted positions int64
        [B][H][n_planted] (1-based)."""
        s = self.shape
        B, H, d = s.batch, s.n_kv_heads, s.head_dim
        G = s.n_q_heads // H
        gen = torch.Generator(device="cpu").manual_seed(seed)
        plen = self.prefix_len.cpu()
        hi = torch.clamp(plen - s.n_recent, min=s.n_sink + 1)        # planted rows stay in J after a step
        u = torch.rand(B, H, n_planted, generator=gen, dtype=torch.float64)
        pos = (s.n_sink + 1 + (u * (hi - s.n_sink).view(B, 1, 1).double()).long()).clamp(max=hi.view(B, 1, 1))
        g_idx = torch.arange(n_planted) % G
        noise = torch.randn(B, H, n_planted, d, generator=gen)
        qh = q.detach().float().cpu().view(B, H, G, d)[:, :, g_idx]   # [B][H][n][d]
        k = (scale * qh + noise).to(torch.bfloat16)
        dev = self.k_cache.device
        bi = torch.arange(B).view(B, 1, 1).expand_as(pos).to(dev)
        hi_ = torch.arange(H).view(1, H, 1).expand_as(pos).to(dev)
        pi = (pos - 1).to(dev)
        self.k_cache[layer][bi, hi_, pi] = k.to(dev)
        self.key_norms[layer][bi, hi_, pi] = k.to(dev).double().pow(2).sum(-1).sqrt()
        return pos

    def step_advance(self, stream=None):
        _C.step_advance(self.shape, self.cache, self._stream(stream))

    def ring_append(self, layer: int, k_new: torch.Tensor, v_new: torch.Tensor, stream=None):
        _C.ring_append(self.shape, self.cache, layer, self._ptr(k_new, torch.bfloat16),
                       self._ptr(v_new, torch.bfloat16), self._stream(stream))

    def append_block(self, layer: int, k: torch.Tensor, v: torch.Tensor, stream=None):
        """k, v: bf16 [B][H][count][d] appended at rows prefix_len[b].. (prefill)."""
        _C.append_block(self.shape, self.cache, layer, k.shape[2], self._ptr(k, torch.bfloat16),
                        self._ptr(v, torch.bfloat16), self._stream(stream))

    def dense_decode(self, layer: int, q: torch.Tensor, out: torch.Tensor,
                     logits: torch.Tensor | None = None, pool: int = 0, stream=None):
        _C.dense_decode(self.shape, self.cache, layer, self._ptr(q, torch.float32),
                        self._ptr(out, torch.float32), self._ptr(logits, torch.float32), pool,
                        self._stream(stream))

    def dense_decode_ex(self, layer: int, q: torch.Tensor, out: torch.Tensor, logits: torch.Tensor | None = None,
                        pool: int = 0, share_sm: bool = False, lse: torch.Tensor | None = None, stream=None,
                        kernel: str | None = None):
        """dense_decode with options: share_sm = leave SM slots to concurrent kernels on
        another stream; lse = natural-log sum-exp per q head; kernel = "tc" (tcgen05 /
        TMEM) or "mma" (mma.sync), default the SFI_DENSE_TC environment choice."""
        flags = (_C.DENSE_SHARE_SM if share_sm else 0) | {None: 0, "tc": _C.DENSE_TC, "mma": _C.DENSE_MMA}[kernel]
        _C.dense_decode_ex(self.shape, self.cache, layer, self._ptr(q, torch.float32),
                           self._ptr(out, torch.float32), self._ptr(lse, torch.float32),
                           self._ptr(logits, torch.float32), pool, flags, self._stream(stream))

    def sparse_decode(self, layer: int, q: torch.Tensor, out: torch.Tensor, stream=None):
        _C.sparse_decode(self.shape, self.cache, layer, self._ptr(q, torch.float32),
                         self._ptr(out, torch.float32), self._stream(stream))

    def fast_decode(self, layer: int, q: torch.Tensor, k_new: torch.Tensor, v_new: torch.Tensor,
                    out: torch.Tensor, prefetch: bool = False, stream=None):
        """One fast step of one layer in ONE launch: ring_append(k_new, v_new) fused
        with sparse_decode. prefetch=True streams the layer's compact rows before
        the PDL wait (valid unless the preceding kernel rebuilt this layer's
        compact cache, include/sfi_b200.h)."""
        _C.fast_decode(self.shape, self.cache, layer, self._ptr(q, torch.float32),
                       self._ptr(k_new, torch.bfloat16), self._ptr(v_new, torch.bfloat16),
                       self._ptr(out, torch.float32), _C.FAST_PREFETCH if prefetch else 0,
                       self._stream(stream))

    def selector(self, layer: int, logits: torch.Tensor, params=None, stream=None):
        _C.selector(self.shape, self.cache, layer, self._ptr(logits, torch.float32),
                    params if params is not None else _C.SelectorParams(), self._stream(stream))

    def prefill_capture(self, layer: int, q_win: torch.Tensor, q_pos: torch.Tensor, out: torch.Tensor,
                        pool: int = 0, stream=None):
        """Prefill tail-window capture: q_win fp32 [B][W][Hq][d] at 1-based positions
        q_pos int32 [B][W] -> pooled logits over J, out fp32 [B][H][W][max_positions]."""
        _C.prefill_capture(self.shape, self.cache, layer, self._ptr(q_win, torch.float32), q_win.shape[1],
                           self._ptr(q_pos, torch.int32), self._ptr(out, torch.float32), pool,
                           self._stream(stream))

    def selector_window(self, layer: int, logits: torch.Tensor, W: int, params=None, stream=None):
        """Selector over a W-row window (prefill): logits fp32 [B][H][W][max_positions]."""
        _C.selector_window(self.shape, self.cache, layer, self._ptr(logits, torch.float32), W,
                           params if params is not None else _C.SelectorParams(), self._stream(stream))

    def selector_fuse(self, layer: int, logits: torch.Tensor, params=None, stream=None) -> torch.Tensor:
        """Head-sharded Selector, phase 1: z_base of this cache's heads, returned as a
        view fp64 [B][H][max_positions] of the workspace (valid until the next
        Selector call on this cache)."""
        ptr, nbytes = _C.selector_fuse(self.shape, self.cache, layer, self._ptr(logits, torch.float32),
                                       params if params is not None else _C.SelectorParams(),
                                       self._stream(stream))
        off = ptr - self.workspace.data_ptr()
        return self.workspace[off:off + nbytes].view(torch.float64).view(
            self.shape.batch, self.shape.n_kv_heads, self.shape.max_positions)

    def selector_finish(self, layer: int, z_all: torch.Tensor, n_shards: int, shard: int, params=None,
                        stream=None):
        """Phase 2 over the all-gathered z_base [n_shards][B][H][max_positions]: soft-NMS,
        cross-head over all heads, top-k of this shard's heads -> sel / n_sel."""
        _C.selector_finish(self.shape, self.cache, layer,
                           params if params is not None else _C.SelectorParams(),
                           self._ptr(z_all, torch.float64), n_shards, shard, self._stream(stream))

    def _C_sel_nccl(self, layer: int, logits: torch.Tensor, params, comm: int, n_shards: int, shard: int,
                    z_all: torch.Tensor, stream=None):
        """KV-head-sharded Selector over an NCCL communicator (sfi_selector_sharded_nccl)."""
        _C.selector_sharded_nccl(self.shape, self.cache, layer, self._ptr(logits, torch.float32),
                                 params if params is not None else _C.SelectorParams(), comm, n_shards, shard,
                                 self._ptr(z_all, torch.float64), self._stream(stream))

    def compact_build(self, layer: int, rebuild_ring: bool = False, stream=None):
        _C.compact_build(self.shape, self.cache, layer, int(bool(rebuild_ring)), self._stream(stream))

    def selector_stages(self, b: int, n_j: int, stream=None):
        return _C.selector_stages(self.shape, self.cache, b, n_j, self._stream(stream))

    def read_errors(self, stream=None):
        """(status, flags, message); clears the device error word."""
        return _C.read_errors(self.cache, self._stream(stream))

    def check_errors(self, stream=None):
        rc, flags, msg = self.read_errors(stream)
        if rc:
            raise _C.SfiError(f"device flags 0x{flags:x}: {msg}")

    @staticmethod
    def last_launch_count() -> int:
        return _C.last_launch_count()


class SlowStepPipeline:
    """Asynchronous slow step (the paper's layer-wise pipeline, PAPER.md:478-495;
    SURVEY §8f-1) over one SfiCache.

    The dense decode of every layer runs on the caller's stream on 65% of the SM
    slots (SFI_DENSE_SHARE_SM; all of them at G = 16); the Selector and the compact build of layer l run
    on an auxiliary stream as soon as layer l's pooled logits exist, on the slots
    the dense kernels leave free, while layers l+1.. stream their KV. The refreshed selection is only read by the next fast step, after `end()`
    joins the streams. Pooled logits go through a ring of `slots` buffers: dense(l)
    waits until the Selector of layer l - slots released its slot."""

    def __init__(self, cache: SfiCache, slots: int = 4, share_sm: bool = True):
        self.c = cache
        self.share_sm = share_sm
        dev = cache.k_cache.device
        s = cache.shape
        self.slots = slots
        self.aux = torch.cuda.Stream(device=dev)
        self.logits = torch.zeros((slots, s.batch, s.n_kv_heads, s.max_positions), dtype=torch.float32,
                                  device=dev)
        self.ev_ready = [torch.cuda.Event() for _ in range(slots)]
        self.ev_free = [torch.cuda.Event() for _ in range(slots)]
        self.used = [False] * slots

    def begin(self):
        self.main = torch.cuda.current_stream()
        self.aux.wait_stream(self.main)  # fork
        self.used = [False] * self.slots

    def layer(self, l: int, q: torch.Tensor, out: torch.Tensor, k_new: torch.Tensor, v_new: torch.Tensor,
              params=None, rebuild_ring: bool = False, dense_events=None):
        """dense_events: optional (start, end) CUDA events recorded on the main stream
        around the dense launch (its in-situ duration beside the aux-stream work)."""
        c, main, s = self.c, self.main, l % self.slots
        if self.used[s]:
            main.wait_event(self.ev_free[s])
        c.ring_append(l, k_new, v_new)
        if dense_events is not None:
            dense_events[0].record(main)
        c.dense_decode_ex(l, q, out, self.logits[s], 0, share_sm=self.share_sm)
        if dense_events is not None:
            dense_events[1].record(main)
        self.ev_ready[s].record(main)
        with torch.cuda.stream(self.aux):
            self.aux.wait_event(self.ev_ready[s])
            c.selector(l, self.logits[s], params)
            c.compact_build(l, rebuild_ring=rebuild_ring)
            self.ev_free[s].record(self.aux)
        self.used[s] = True

    def end(self):
        self.main.wait_stream(self.aux)  # join: the next fast step reads the new compact rows


class StepExecutor:
    """The C++ decode executor (include/sfi/decode.hpp, executor.cpp) over one
    SfiCache: whole decode steps of all layers — fast (advance + one fused K4
    launch per layer) or slow (the layer-wise asynchronous pipeline: dense on the
    main stream, Selector + compact on an aux stream through a `slots`-deep
    pooled-logit ring, one completion barrier; `priorities=1` makes the main
    stream high- and the aux stream lowest-priority, kept as graph node
    priorities — measured slower) — enqueued from C++, capturable
    once per kind into a CUDA graph and replayed with no host work.

    q, out: fp32 [L][B][Hq][d]; k_new, v_new: bf16 [L][B][H][d] (views with any
    per-layer stride, e.g. rows of one packed [L][q | k | v] buffer)."""

    def __init__(self, cache: SfiCache, selector=None, slots: int = 2, share_sm: bool = True, stream=None,
                 priorities: int = 0):
        self.c = cache
        self.stream = stream if stream is not None else torch.cuda.Stream(device=cache.k_cache.device)
        s = cache.shape
        self.logits = torch.zeros((slots, s.batch, s.n_kv_heads, s.max_positions), dtype=torch.float32,
                                  device=cache.k_cache.device)
        self.x = _C.DecodeExecutor(cache.shape, cache.cache, self.stream.cuda_stream,
                                   selector if selector is not None else _C.SelectorConfig(), slots, share_sm,
                                   self.logits.data_ptr(), priorities)

    @staticmethod
    def _stride(t: torch.Tensor) -> int:
        return t.stride(0) * t.element_size()

    def _args(self, q, k_new, v_new, out):
        for t in (q, k_new, v_new, out):
            if not t.is_cuda or not t[0].is_contiguous():
                raise ValueError("step buffers: CUDA tensors with contiguous layers")
        return (q.data_ptr(), k_new.data_ptr(), v_new.data_ptr(), out.data_ptr(), self._stride(q),
                self._stride(k_new), self._stride(out))

    def step(self, slow: bool, q, k_new, v_new, out, rebuild_ring: bool = False, wait_before=(), record_after=(),
             origin=None, record_before_attention=(), aux_events=((), (), ())):
        """Enqueue one step after the work on `origin` (a torch stream; default: the
        executor's stream). wait_before / record_after / record_before_attention:
        per-layer torch.cuda.Events (the last two bracket each layer's attention
        launch on the main stream); aux_events: three per-layer lists recorded on the
        aux stream of a slow step (before the Selector, after it, after the compact
        rebuild)."""
        if k_new.stride(0) * k_new.element_size() != self._stride(v_new):
            raise ValueError("k_new / v_new layer strides differ")
        ev = lambda es: [e.cuda_event if e is not None else 0 for e in es]  # noqa: E731
        self.x.step(slow, *self._args(q, k_new, v_new, out), rebuild_ring, ev(wait_before), ev(record_after), False,
                    0 if origin is None else origin.cuda_stream, ev(record_before_attention),
                    [x for es in aux_events for x in ev(es)])

    def capture(self, slow: bool, q, k_new, v_new, out, rebuild_ring: bool = False):
        self.x.step(slow, *self._args(q, k_new, v_new, out), rebuild_ring, [], [], True, 0)

    def replay(self, slow: bool):
        self.x.replay(slow)

    def logits_slot(self, layer: int) -> torch.Tensor:
        """Layer `layer`'s pooled logits after a slow step (until layer + slots reuses the slot)."""
        return self.logits[layer % self.logits.shape[0]]

"""SFI decode-attention hot-path benchmark (BASELINE.json metric: SFI decode
tokens/s at 32K-256K context; fast/slow step us; HBM GB/s vs peak).

A step = one SFI decode step of the whole hot path for a batch of requests:
  advance the prefix, then for every layer
    fast: ring append (K3) + sparse decode over the compact cache (K4)
    slow: ring append (K3) + dense decode with pooled logits (K1)
          + Selector (K2) + compact build (K3)
following a seeded schedule (step 0 slow; triggers Bernoulli(1/24); forced at
t_max = 64, scheduler.cpp:93-99). Default workload = configs[1] (C2):
Qwen3-8B-shaped attention (32 q / 8 kv heads, d = 128, 36 layers), batch 8,
32K context, CacheLimits defaults (sink 4, selected 2048, recent 256).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c1|c2|c3]
    python bench.py --impl reference ...   # the reference CPU path on the host cores

Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (workload, n_layers, Hq, H, batch, context, n_sink, k_budget, n_recent)
    "c1": ("Qwen3-0.6B-shaped attention, batch 1, 8K", 28, 16, 8, 1, 8192, 4, 512, 64),
    "c2": ("Qwen3-8B-shaped attention, batch 8, 32K", 36, 32, 8, 8, 32768, 4, 2048, 256),
    "c3": ("Qwen3-32B-shaped attention, batch 4, 128K", 64, 64, 8, 4, 131072, 4, 2048, 256),
    "c4": ("Qwen3-235B-shaped attention, batch 1, 256K", 94, 64, 4, 1, 262144, 4, 2048, 256),
}
# multi-GPU partitioning per config: "dp" = independent request
# batches per GPU (weak scaling); "heads" = KV-head sharding of ONE batch
# (strong scaling, z_base all-gather in the Selector)
SHARDING = {"c1": "dp", "c2": "dp", "c3": "heads", "c4": "seq"}
# steps per timed window when --steps is not given (C1 256-step schedule,
# C2 512 steps, C3/C4 64-step windows); the driver passes --steps explicitly
DEFAULT_STEPS = {"c1": 256, "c2": 512, "c3": 64, "c4": 64}
HEAD_DIM = 128
T_MAX = 64
P_TRIGGER = 1.0 / 24.0


def metric_name(cfg_name: str) -> str:
    name, _, _, _, _, ctx = CONFIGS[cfg_name][:6]
    return f"SFI decode tokens/s ({ctx // 1024}K ctx, {name.split(',')[0]}, batch {CONFIGS[cfg_name][4]})"


def parallelism(cfg_name: str, world: int) -> str:
    mode = SHARDING[cfg_name] if world > 1 else "single"
    return {"heads": f"kv-head sharded x{world} (one batch; z_base of every slow-step layer all-gathered)",
            "seq": f"sequence sharded x{world} (LSE-merged attention partials; Selector statistics, soft-NMS "
                   "edges and top-k candidates all-gathered)",
            "dp": f"dp{world} (independent request batches per GPU)"}.get(mode, "1 GPU")


def config_dict(cfg_name: str, world: int) -> dict:
    """The workload, identical in both arms (the reference arm times the same
    config on the host cores)."""
    name, n_layers, Hq, H, B, ctx, ns, K, R = CONFIGS[cfg_name]
    return {"workload": f"{name} ({cfg_name.upper()})", "layers": n_layers, "q_heads": Hq, "kv_heads": H,
            "head_dim": HEAD_DIM, "batch": B * (world if SHARDING[cfg_name] == "dp" and world > 1 else 1),
            "context": ctx, "n_sink": ns, "k_budget": K, "n_recent": R,
            "schedule": f"step 0 slow; seeded triggers p=1/24; forced at t_max={T_MAX}",
            "parallelism": parallelism(cfg_name, world),
            "l2": "inputs larger than L2 (KV cache >= 1 GB per layer group)"}


def schedule(n_steps: int, seed: int) -> list[bool]:
    """True = slow. Step 0 slow; afterwards slow iff the previous token was a
    trigger (Bernoulli(1/24)) or steps_since_slow + 1 >= t_max."""
    rng = np.random.default_rng(seed)
    out, since, trig = [], 0, True
    for _ in range(n_steps):
        slow = trig or since + 1 >= T_MAX
        out.append(slow)
        since = 0 if slow else since + 1
        trig = bool(rng.random() < P_TRIGGER)
    return out


def peaks() -> dict:
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return {"hbm_gbs": float(d["hbm_gbs"]), "source": "measured"}
    except Exception:
        return {"hbm_gbs": 6650.0, "source": "fallback"}


class ClockSampler:
    """Samples SM clock and throttle reasons with NVML during the timed region."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
        0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, index: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and bit != 0x1:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.005)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv:
            self.t.join()

    def summary(self) -> dict:
        med = statistics.median(self.samples) if self.samples else None
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


# ---------------------------------------------------------------------------
# GPU arm

class Workload:
    def __init__(self, cfg_name: str, steps_total: int, device, world: int = 1, layers: int = 0,
                 sync_slow: bool = False, inputs: str = "iid", backend: str = "nccl"):
        import torch

        import paper_2603_12038_b200 as sfi

        (self.name, self.L, self.Hq, self.H, self.B, self.ctx, self.ns, self.K,
         self.R) = CONFIGS[cfg_name]
        if layers:
            self.L = layers
        self.cfg_name = cfg_name
        self.G = self.Hq // self.H
        self.Lmax = self.ctx + steps_total + 64
        self.torch = torch
        self.mode = SHARDING[cfg_name] if world > 1 else "single"
        self.world = world
        fill_len = self.ctx
        # exchange of the sharded configs (SFI_SEQ_EXCHANGE): "nccl" (default on the nccl
        # backend) = the C ABI's in-call ncclAllGather on torch's communicator
        # (sfi_selector_sharded_nccl / sfi_merge_partials_nccl / sfi_seq_selector_nccl);
        # "allgather" = torch.distributed all-gathers (the gloo default); "peer" = CUDA-IPC
        # peer memory (opt-in: only the one-GPU two-process form has run)
        xch = os.environ.get("SFI_SEQ_EXCHANGE", "nccl" if backend == "nccl" else "allgather")
        self.exchange = xch if world > 1 else "none"
        self.peer = world > 1 and self.L >= 2 and xch == "peer"
        nccl = world > 1 and xch == "nccl"
        if self.mode == "heads":
            from paper_2603_12038_b200.sharded import HeadShardedSfi

            mk = lambda **kw: HeadShardedSfi(self.L, self.B, self.H, self.Hq, HEAD_DIM, self.Lmax, self.ns,  # noqa
                                             self.K, self.R, device=device, **kw)
            try:
                self.drv = mk(peer=self.peer, nccl=nccl)
            except Exception as e:  # pragma: no cover - every rank votes in the peer setup (sharded.agree)
                print(f"{xch} exchange unavailable ({e}); using torch all-gather", file=sys.stderr)
                self.peer, self.exchange = False, "allgather"
                self.drv = mk()
            self.H, self.Hq = self.drv.local_heads, self.drv.local_heads * self.G  # this rank's heads
        elif self.mode == "seq":
            from paper_2603_12038_b200.sharded import SeqShardedSfi

            mk = lambda **kw: SeqShardedSfi(self.L, self.B, self.H, self.Hq, HEAD_DIM, self.Lmax, self.ctx,  # noqa
                                            self.ns, self.K, self.R, device=device, **kw)
            try:
                self.drv = mk(peer=self.peer, nccl=nccl)
            except Exception as e:  # pragma: no cover
                print(f"{xch} exchange unavailable ({e}); using torch all-gather", file=sys.stderr)
                self.peer, self.exchange = False, "allgather"
                self.drv = mk()
            fill_len = min(self.drv.cap, self.ctx - self.drv.base)  # this rank's positions
        else:
            self.drv = sfi.SfiCache(self.L, self.B, self.H, self.Hq, HEAD_DIM, self.Lmax, self.ns,
                                    self.K, self.R, device=device)
        self.cache = self.drv if self.mode in ("single", "dp") else self.drv.cache
        # tokens produced per step by the whole job, per rank's share of it
        self.job_tokens = self.B * (world if self.mode == "dp" else 1)
        self.params = sfi.SelectorParams()
        t = torch
        g = t.Generator(device="cpu").manual_seed(2027)
        L, B, H, Hq, d = self.L, self.B, self.H, self.Hq, HEAD_DIM
        # per-layer step inputs, resident in HBM (q fp32 from the projection; new K/V bf16),
        # packed per layer [q | k_new | v_new] so one copy moves a layer group's inputs
        qb, kb = B * Hq * d * 4, B * H * d * 2
        self.io = t.empty(L, qb + 2 * kb, dtype=t.uint8, device=device)
        self.q = self.io[:, :qb].view(t.float32).view(L, B, Hq, d)
        self.k_new = self.io[:, qb:qb + kb].view(t.bfloat16).view(L, B, H, d)
        self.v_new = self.io[:, qb + kb:].view(t.bfloat16).view(L, B, H, d)
        self.q.copy_(t.randn(L, B, Hq, d, generator=g))
        self.k_new.copy_(t.randn(L, B, H, d, generator=g).bfloat16())
        self.v_new.copy_(t.randn(L, B, H, d, generator=g).bfloat16())
        self.out = t.zeros(L, B, Hq, d, device=device)
        self.logits = self.cache.pooled_logits
        drv = self.drv
        # 1 GPU / dp: whole steps through the C++ decode executor (include/sfi/decode.hpp):
        # the asynchronous slow step (Selector + compact of layer i on an aux stream behind
        # the dense decode of layers i+1..) and graph-captured steps
        self.pipe = None
        self.exec = None
        if self.mode in ("single", "dp") and not sync_slow:
            from paper_2603_12038_b200.device import StepExecutor

            self.exec = StepExecutor(self.cache, slots=int(os.environ.get("SFI_EXEC_SLOTS", "2")),
                                     priorities=int(os.environ.get("SFI_EXEC_PRIO", "0")))
        self.cache.fill_synthetic(seed=2026 + 1, length=fill_len)
        self.set_lengths(self.ctx)
        if inputs == "peaked" and self.mode in ("single", "dp", "heads"):
            # 32 planted positions per (b, KV head) with k = 3 q + noise
            for l in range(L):
                self.cache.plant_peaked(l, self.q[l], n_planted=32, scale=3.0, seed=2026 + l)
        # initial slow step (untimed): dense + Selector + compact incl. the ring
        self.step(slow=True, rebuild_ring=True)
        t.cuda.synchronize()
        drv.check_errors()
        # exercise the fast path once eagerly (same prefix: undo its advance)
        self.step(slow=False)
        self.set_lengths(self.ctx + 1)
        t.cuda.synchronize()
        drv.check_errors()

    def set_lengths(self, L: int):
        self.drv.set_lengths([L] * self.B, [self.ns] * self.B)

    def step(self, slow: bool, rebuild_ring: bool = False, io=None):
        """One decode step of all layers through the mode's driver: SfiCache (1 GPU /
        dp), HeadShardedSfi (z_base all-gather in the Selector) or SeqShardedSfi
        (LSE-merged attention partials, sharded Selector statistics). `io`: the
        end-to-end variant's per-layer host copies (HostIO)."""
        d = self.drv
        if self.exec is not None:
            origin = self.torch.cuda.current_stream()
            if io is not None:
                io.begin()
            wb, ra = io.hook_events() if io is not None else ((), ())
            self.exec.step(slow, self.q, self.k_new, self.v_new, self.out, rebuild_ring, wb, ra, origin=origin)
            if io is not None:
                io.copy_outputs()
                io.end()
            return
        if io is not None:
            io.begin()
        d.step_advance()
        pipe = self.pipe if (slow and self.pipe is not None) else None
        if pipe is not None:
            pipe.begin()
        for l in range(self.L):
            if io is not None:
                io.before(l)
            if pipe is not None:  # dense on this stream, Selector + compact on the aux stream
                pipe.layer(l, self.q[l], self.out[l], self.k_new[l], self.v_new[l], self.params, rebuild_ring)
            elif slow:
                d.ring_append(l, self.k_new[l], self.v_new[l])
                d.dense_decode(l, self.q[l], self.out[l], self.logits, 0)
                d.selector(l, self.logits, self.params)
                d.compact_build(l, rebuild_ring=rebuild_ring)
            else:
                # ONE launch: ring append fused with the sparse decode; the
                # compact rows of layer l are not written by the preceding
                # kernel, so they stream before the PDL wait
                d.fast_decode(l, self.q[l], self.k_new[l], self.v_new[l], self.out[l], prefetch=True)
            if io is not None:
                io.after(l)
        if pipe is not None:
            pipe.end()
        if io is not None:
            io.end()

    # the attention kernels alone (per-kernel timing), no exchange
    def fast_kernel(self, l: int):
        if self.mode == "seq":
            self.drv.fast_partial(l, self.q[l], self.k_new[l], self.v_new[l], prefetch=True)
        else:
            self.cache.fast_decode(l, self.q[l], self.k_new[l], self.v_new[l], self.out[l], prefetch=True)

    def dense_kernel(self, l: int):
        if self.mode == "seq":
            self.drv.dense_partial(l, self.q[l], self.logits)
        else:
            self.cache.dense_decode(l, self.q[l], self.out[l], self.logits, 0)

    def launches(self, slow: bool) -> int:
        """Our kernels per step (collectives' own kernels not counted)."""
        xch = 3 if getattr(self, "peer", False) else 2  # partial (+ publish) + merge
        if not slow:  # advance + one fused launch per layer (+ the LSE merge when sequence-sharded)
            return 1 + self.L * (xch if self.mode == "seq" else 1)
        if self.mode == "seq":  # append (last rank), dense + merge, Selector 2 stats + finish 3 + pick 3
            # (+ 3 publishes and 4 peer gathers over peer memory), compact
            return 1 + self.L * (1 + xch + (15 if getattr(self, "peer", False) else 8) + 1)
        if self.mode == "heads":  # append, dense, Selector fuse + refine + top-k, compact (+ copy, publish, gather)
            return 1 + self.L * (6 + (3 if getattr(self, "peer", False) else 0))
        return 1 + self.L * 7  # append, dense, Selector pw + coef + z + top-k, compact

    def shard_frac(self) -> float:  # this rank's share of a layer's rows (sequence shards)
        return 1.0 / self.world if self.mode == "seq" else 1.0

    # algorithmic bytes of one launch
    def bytes_sparse(self) -> float:
        # S rows of K+V (the current token's from k_new/v_new), q in, o out, and
        # the append: paged + ring row of K and V plus the fp64 norm
        S = self.R + self.ns + self.K
        return (self.B * self.H * (S * 4 * HEAD_DIM * self.shard_frac() + 2 * 4 * HEAD_DIM + 8)
                + 2 * self.B * self.Hq * HEAD_DIM * 4)

    def bytes_slow_layer(self, Lcur: int) -> float:
        """A slow-step layer's algorithmic bytes: dense KV + pooled
        logits write (bytes_dense), the Selector's inputs (fp32 logits + fp64 norms
        over J), the compact gather (sink + selected rows read and written, plus the
        ring rebuild is not counted: the timed steps do not rebuild it) and the append."""
        rl = min(self.R, Lcur - self.ns)
        nj = (Lcur - rl - self.ns) * self.shard_frac()
        return (self.bytes_dense(Lcur) + self.B * self.H * nj * (4 + 8)
                + self.B * self.H * (self.ns + self.K) * 4 * HEAD_DIM * 2 + self.B * self.H * (2 * 4 * HEAD_DIM + 8))

    def bytes_dense(self, Lcur: int) -> float:
        rl = min(self.R, Lcur - self.ns)
        nj = Lcur - rl - self.ns
        return ((self.B * self.H * Lcur * 4 * HEAD_DIM + self.B * self.H * nj * 4) * self.shard_frac()
                + 2 * self.B * self.Hq * HEAD_DIM * 4)


class HostIO:
    """End-to-end step I/O: every step copies its inputs (q fp32, new K/V bf16) from
    pinned host memory and its output back to pinned host memory, in groups of
    layers on a copy stream ordered with the compute stream by events — a group's
    inputs land while the previous group computes and its output returns while the
    next group computes (few, large copies: each copy node costs microseconds)."""

    def __init__(self, wl: Workload, group: int | None = None):
        t = wl.torch
        if group is None:  # >= 6 layers and >= ~512 KB of inputs per copy group
            per_layer = (wl.q[0].numel() * 4 + wl.k_new[0].numel() * 4)
            group = max(6, -(-(512 << 10) // per_layer))
            group = int(os.environ.get("SFI_BENCH_IO_GROUP", group))
        self.t, self.wl = t, wl
        self.cs = t.cuda.Stream()
        pin = lambda x: t.empty_like(x, device="cpu").pin_memory()  # noqa: E731
        self.ioh, self.oh = pin(wl.io), pin(wl.out)  # [L][q | k_new | v_new] bytes, [L] outputs
        self.ioh.copy_(wl.io)
        # one-layer groups at both ends: the first inputs and the last output are
        # the only copies the compute cannot hide
        cuts = [0] + ([1] if wl.L > 2 else []) + list(range(1 + group, wl.L - 1, group)) + \
            ([wl.L - 1] if wl.L > 2 else []) + [wl.L]
        cuts = sorted(set(c for c in cuts if 0 <= c <= wl.L))
        self.groups = [(a, b) for a, b in zip(cuts[:-1], cuts[1:]) if b > a]
        self.ev_in = [t.cuda.Event() for _ in self.groups]
        self.ev_out = [t.cuda.Event() for _ in self.groups]
        for e in self.ev_in + self.ev_out:  # create the CUDA events now (the executor records / waits on them)
            e.record()
        self.h2d = wl.q.numel() * 4 + wl.k_new.numel() * 2 + wl.v_new.numel() * 2
        self.d2h = wl.out.numel() * 4

    def begin(self):
        t, wl, cs = self.t, self.wl, self.cs
        self.main = t.cuda.current_stream()
        cs.wait_stream(self.main)  # fork
        with t.cuda.stream(cs):
            for gi, (l0, l1) in enumerate(self.groups):
                wl.io[l0:l1].copy_(self.ioh[l0:l1], non_blocking=True)  # q, k_new, v_new of the group
                self.ev_in[gi].record(cs)

    def before(self, l: int):
        for gi, (l0, _) in enumerate(self.groups):
            if l == l0:
                self.main.wait_event(self.ev_in[gi])

    def after(self, l: int):
        for gi, (l0, l1) in enumerate(self.groups):
            if l == l1 - 1:
                self.ev_out[gi].record(self.main)
                with self.t.cuda.stream(self.cs):
                    self.cs.wait_event(self.ev_out[gi])
                    self.oh[l0:l1].copy_(self.wl.out[l0:l1], non_blocking=True)

    def hook_events(self):
        """Per-layer events for the C++ executor: the main stream waits for a group's
        inputs before its first layer and marks its last layer's output."""
        wb, ra = [None] * self.wl.L, [None] * self.wl.L
        for gi, (l0, l1) in enumerate(self.groups):
            wb[l0] = self.ev_in[gi]
            ra[l1 - 1] = self.ev_out[gi]
        return wb, ra

    def copy_outputs(self):
        with self.t.cuda.stream(self.cs):
            for gi, (l0, l1) in enumerate(self.groups):
                self.cs.wait_event(self.ev_out[gi])
                self.oh[l0:l1].copy_(self.wl.out[l0:l1], non_blocking=True)

    def end(self):
        self.main.wait_stream(self.cs)  # join: the step ends when its output is on the host


def time_kernel(wl: Workload, which: str, iters: int) -> float:
    """Average device duration (ms) of one decode launch, isolated: `iters`
    launches (cycling the layers) queued back to back between two CUDA events on
    the launching stream, so host launch overhead is not in the figure."""
    t = wl.torch
    s = t.cuda.current_stream()
    fn = wl.fast_kernel if which == "sparse" else wl.dense_kernel
    for l in range(min(2, wl.L)):  # warm
        fn(l)
    t.cuda.synchronize()
    a, b = t.cuda.Event(enable_timing=True), t.cuda.Event(enable_timing=True)
    a.record(s)
    for i in range(iters):
        fn(i % wl.L)
    b.record(s)
    t.cuda.synchronize()
    return a.elapsed_time(b) / iters


def time_graph(g, reps: int, stream=None) -> float:
    """ms per replay of a captured step (a torch CUDAGraph or the executor's replay
    callable), back to back between two events on the stream it replays on
    (default: the current stream)."""
    t = __import__("torch")
    if stream is None:
        stream = t.cuda.current_stream()
    run = g if callable(g) else g.replay
    run()
    t.cuda.synchronize()
    a, b = t.cuda.Event(enable_timing=True), t.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(reps):
        run()
    b.record(stream)
    t.cuda.synchronize()
    return a.elapsed_time(b) / reps


def fast_grid(wl: Workload) -> int:
    """CTAs of one fused fast-step launch (fast_decode.cu fast_cluster_size)."""
    slices, c = wl.B * wl.H, 1
    tiles = -(-wl.R // 64) + -(-(wl.ns + wl.K) // 64)
    if 2 <= tiles <= 16 and slices * tiles <= 2 * 148:  # small slices: one tile per CTA
        return slices * tiles
    while c < 8 and slices * c <= 148:
        c *= 2
    if c == 8 and slices * 32 <= 148:
        c = 16
    return slices * c


def launch_floor_ms(wl: Workload) -> float | None:
    """Per-layer launch floor of the fast step: a CUDA graph of 1 + L empty
    kernels (sfi_launch_floor) with the fused fast step's PDL protocol and grid,
    replayed back to back; ms per launch."""
    import paper_2603_12038_b200 as sfi

    t = wl.torch
    try:
        g = t.cuda.CUDAGraph()
        s = t.cuda.Stream()
        with t.cuda.stream(s):
            sfi._C.launch_floor(2, fast_grid(wl), s.cuda_stream)  # warm
        t.cuda.synchronize()
        with t.cuda.graph(g):
            sfi._C.launch_floor(1 + wl.L, fast_grid(wl), t.cuda.current_stream().cuda_stream)
        return time_graph(g, 16, t.cuda.current_stream()) / (1 + wl.L)
    except Exception:
        return None


def time_selector(wl: Workload, iters: int) -> tuple[float, float]:
    """Selector and compact build per layer, isolated (queued back to back)."""
    t = wl.torch
    s = t.cuda.current_stream()
    c = wl.cache
    wl.drv.selector(0, wl.logits, wl.params)
    t.cuda.synchronize()
    a, b, e = (t.cuda.Event(enable_timing=True) for _ in range(3))
    a.record(s)
    for i in range(iters):
        wl.drv.selector(i % wl.L, wl.logits, wl.params)
    b.record(s)
    for i in range(iters):
        c.compact_build(i % wl.L)
    e.record(s)
    t.cuda.synchronize()
    return a.elapsed_time(b) / iters, b.elapsed_time(e) / iters


def time_dense_in_situ(wl: Workload) -> tuple[float | None, float | None]:
    """K1 as it runs inside the timed slow step: one eager asynchronous slow step
    through the C++ executor (dense on the main stream at the pipeline's share grid,
    Selector + compact of the earlier layers concurrently on the aux stream), with
    the executor's per-layer hooks recording events on the main stream right before
    each dense launch and right after it. Returns (mean dense launch duration, mean
    per-layer main-chain period incl. the ring append and the logit-slot waits),
    both over layers 2.. (layers 0-1 run with an idle aux stream)."""
    if wl.exec is None:
        return None, None
    t = wl.torch
    before = [t.cuda.Event(enable_timing=True) for _ in range(wl.L)]
    after = [t.cuda.Event(enable_timing=True) for _ in range(wl.L)]
    for e in before + after:
        e.record()
    wl.set_lengths(wl.ctx)
    t.cuda.synchronize()
    wl.exec.step(True, wl.q, wl.k_new, wl.v_new, wl.out, False, (), after, record_before_attention=before)
    t.cuda.synchronize()
    launch = [before[i].elapsed_time(after[i]) for i in range(2, wl.L)]
    period = [after[i - 1].elapsed_time(after[i]) for i in range(2, wl.L)]
    return (float(np.mean(launch)), float(np.mean(period))) if launch else (None, None)


def traffic_for(kernel: str, cfg_name: str):
    """DRAM bytes (read + write) per launch of `kernel` at `cfg_name` from the
    committed ncu --set full captures (profiles/r02/traffic.json, else r01's C2
    figures); None when no capture of that kernel at that config exists."""
    for rnd in ("r02", "r01"):
        try:
            with open(os.path.join(ROOT, "profiles", rnd, "traffic.json")) as f:
                t = json.load(f)
        except Exception:
            continue
        e = t.get(cfg_name, {}).get(kernel) if cfg_name in t else (t.get(kernel) if cfg_name == "c2" else None)
        if e:
            return e["dram_read_bytes"] + e["dram_write_bytes"], f"profiles/{rnd}/traffic.json"
    return None, f"no ncu capture of {kernel} at {cfg_name}"


# C5 (BASELINE configs[4]): long-CoT generation, 2K prefill + 32K generated tokens on
# Qwen3-8B attention shapes, batch 8; SFI (K = 2048) across the generation vs full-KV
# dense decode; the refresh budget t_max swept through the seeded schedule's slow fraction
C5 = dict(layers=36, q_heads=32, kv_heads=8, batch=8, prefill=2048, generated=32768, n_sink=4, k_budget=2048,
          n_recent=256)
C5_TMAX = (16, 32, 64, 128)


def c5_slow_fraction(t_max: int, steps: int, seed: int = 2031) -> float:
    """Slow steps / steps of the seeded schedule over a whole generation (step 0 slow;
    triggers Bernoulli(1/24), forced at t_max; scheduler.cpp:93-99)."""
    rng = np.random.default_rng(seed)
    since, trig, n = 0, True, 0
    for _ in range(steps):
        slow = trig or since + 1 >= t_max
        n += slow
        since = 0 if slow else since + 1
        trig = bool(rng.random() < P_TRIGGER)
    return n / steps


def run_c5(dev, k_budget: int | None = None, batch: int | None = None, dense: bool = True) -> dict:
    """The C5 line: per context point of the generation (2K, 10K, 18K, 26K, 34K) the
    executor's fast and slow steps and a full-KV dense step (append + K1 over the
    whole cache, every layer) are replayed from CUDA graphs; a schedule's time per
    token is (1 - f) fast + f slow, averaged over the generation (trapezoid in
    context). scripts/sweep_c5.py calls it per (K, batch)."""
    import torch

    import paper_2603_12038_b200 as sfi
    from paper_2603_12038_b200.device import StepExecutor

    c5 = C5
    L, Hq, H, d = c5["layers"], c5["q_heads"], c5["kv_heads"], HEAD_DIM
    B = batch or c5["batch"]
    ns, K, R = c5["n_sink"], k_budget or c5["k_budget"], c5["n_recent"]
    ctxs = [c5["prefill"] + i * c5["generated"] // 4 for i in range(5)]
    cache = sfi.SfiCache(L, B, H, Hq, d, ctxs[-1] + 64, ns, K, R, device=dev)
    cache.fill_synthetic(seed=2031, length=ctxs[-1])
    g = torch.Generator().manual_seed(2031)
    q = torch.randn(L, B, Hq, d, generator=g).to(dev)
    kn = torch.randn(L, B, H, d, generator=g).bfloat16().to(dev)
    vn = torch.randn(L, B, H, d, generator=g).bfloat16().to(dev)
    out = torch.zeros(L, B, Hq, d, device=dev)
    x = StepExecutor(cache, slots=2)
    st = x.stream
    fast_ms, slow_ms, dense_ms = {}, {}, {}

    def at(ctx):
        cache.set_lengths([ctx] * B, [ns] * B)
        torch.cuda.synchronize()

    for ctx in ctxs:
        at(ctx)
        x.step(True, q, kn, vn, out, rebuild_ring=True)  # selection + compact cache at this context
        x.step(False, q, kn, vn, out)
        st.synchronize()
        at(ctx)
        x.capture(False, q, kn, vn, out)
        x.capture(True, q, kn, vn, out)
        at(ctx)
        fast_ms[ctx] = time_graph(lambda: x.replay(False), 8, st)
        at(ctx)
        slow_ms[ctx] = time_graph(lambda: x.replay(True), 3, st)
        cache.check_errors()
    if dense:
        gd = torch.cuda.CUDAGraph()
        with torch.cuda.stream(st):
            at(ctxs[0])

            def dense_step():
                cache.step_advance()
                for l in range(L):
                    cache.ring_append(l, kn[l], vn[l])
                    cache.dense_decode(l, q[l], out[l])

            dense_step()  # eager once (kernel attributes), then capture
            st.synchronize()
            with torch.cuda.graph(gd, stream=st):
                dense_step()
        for ctx in ctxs:
            at(ctx)
            with torch.cuda.stream(st):  # a torch graph replays on the current stream
                dense_ms[ctx] = time_graph(gd, 3, st)
        cache.check_errors()

    def gen_avg(per):  # mean ms per step over a generation uniform in context
        ys = [per[c] for c in ctxs]
        return float(np.trapezoid(ys, ctxs) / (ctxs[-1] - ctxs[0]))

    dense_avg = gen_avg(dense_ms) if dense else None
    rows = []
    for t in C5_TMAX:
        f = c5_slow_fraction(t, c5["generated"])
        avg = gen_avg({c: (1 - f) * fast_ms[c] + f * slow_ms[c] for c in ctxs})
        rows.append({"t_max": t, "slow_fraction": round(f, 4), "tokens_per_s": B / (avg / 1e3),
                     "speedup_vs_full_kv": dense_avg / avg if dense else None})
    head = next(r for r in rows if r["t_max"] == T_MAX)
    del x, cache
    _release()
    return {"metric": f"SFI decode tokens/s (C5 long-CoT: {c5['prefill'] // 1024}K prefill + "
                      f"{c5['generated'] // 1024}K generated, Qwen3-8B-shaped attention, batch {B})",
            "value": head["tokens_per_s"], "unit": "tokens/s", "n_gpus": 1, "higher_is_better": True,
            "full_kv_dense_tokens_per_s": B / (dense_avg / 1e3) if dense else None,
            "speedup_vs_full_kv": head["speedup_vs_full_kv"],
            "t_max": T_MAX, "sweep": rows,
            "per_context_ms": {str(c): {"fast": fast_ms[c], "slow": slow_ms[c], "full_kv_dense": dense_ms.get(c)}
                               for c in ctxs},
            "config": {"workload": "Qwen3-8B-shaped attention, long-CoT generation (C5)", "layers": L,
                       "q_heads": Hq, "kv_heads": H, "head_dim": d, "batch": B, "prefill": c5["prefill"],
                       "generated": c5["generated"], "n_sink": ns, "k_budget": K, "n_recent": R,
                       "contexts": ctxs},
            "timing": "CUDA-graph replays of the executor's fast / slow steps and of a full-KV dense step at each "
                      "context point (CUDA events on the replay stream); the schedule mixes them by its seeded slow "
                      "fraction over the 32K generated tokens; per-K sweep: scripts/sweep_c5.py"}


def _release(*objs):
    import gc

    import torch
    for o in objs:
        if isinstance(o, dict):
            for g in o.values():
                try:
                    g.reset()
                except Exception:
                    pass
    gc.collect()
    torch.cuda.synchronize()
    torch.cuda.empty_cache()


def run_config(cfg_name: str, args, ctx: dict, full: bool) -> dict:
    """One workload end to end on this rank: setup, warm-up, K timed steps (max over
    ranks), the end-to-end variant and the per-kernel timings. `full` adds the e2e
    and CPU-baseline legs (the headline config)."""
    import torch
    import torch.distributed as dist

    world, rank, local, dev = ctx["world"], ctx["rank"], ctx["local"], ctx["dev"]
    max_over_ranks = ctx["max_over_ranks"]
    W = args.warmup
    K = args.steps if args.steps else DEFAULT_STEPS[cfg_name]
    sched = schedule(W + K + 1, seed=2026 + 1)[1:]  # step 0 of the schedule is the setup slow step
    wl = Workload(cfg_name, W + K + 8, dev, world, args.layers, args.sync_slow, inputs=args.inputs,
                  backend=args.backend)
    c = wl.cache
    use_graph = not args.no_graph
    graphs = {}
    graph_note = None
    # the stream the timed steps run on: the C++ executor's own stream (its graphs keep
    # their node priorities), else torch's current stream
    stream = wl.exec.stream if wl.exec is not None else torch.cuda.current_stream()
    if use_graph:
        # both paths already ran eagerly in setup (kernel attributes, driver entry
        # points); capture records without executing, so prefix_len is untouched
        try:
            for slow in (False, True):
                if wl.exec is not None:
                    wl.exec.capture(slow, wl.q, wl.k_new, wl.v_new, wl.out)
                    graphs[slow] = (lambda s_=slow: wl.exec.replay(s_))
                else:
                    g = torch.cuda.CUDAGraph()
                    with torch.cuda.graph(g):
                        wl.step(slow)
                    graphs[slow] = g
            torch.cuda.synchronize()
        except Exception as ex:  # e.g. a collective backend that cannot be captured
            use_graph, graphs = False, {}
            graph_note = f"graph capture failed ({type(ex).__name__}); eager launches"
            torch.cuda.synchronize()
            wl.set_lengths(wl.ctx + 1)

    def run(slow: bool):
        if use_graph:
            g = graphs[slow]
            g() if callable(g) else g.replay()
        else:
            with torch.cuda.stream(stream):
                wl.step(slow)

    for i in range(W):
        run(sched[i])
    torch.cuda.synchronize()
    wl.drv.check_errors()

    timed = sched[W:W + K]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        e0.record(stream)
        for slow in timed:
            run(slow)
        e1.record(stream)
        torch.cuda.synchronize()
    ms = max_over_ranks(e0.elapsed_time(e1))
    if world > 1:
        dist.barrier()
    wl.drv.check_errors()
    n_slow = sum(timed)
    value = wl.job_tokens * K / (ms / 1e3)

    # ---- end to end through the public API with host buffers ----
    e2e = None
    ge = {}
    if full and not args.no_e2e:
        io = HostIO(wl)
        if use_graph:
            for slow in (False, True):
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g):
                    wl.step(slow, io=io)
                ge[slow] = g
            torch.cuda.synchronize()
        sched_e = sched[W:W + K]  # the same schedule as the device-resident timing
        wl.set_lengths(wl.ctx + 1)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        cur = torch.cuda.current_stream()  # torch's graphs replay on the current stream
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(cur)
        for slow in sched_e:
            if use_graph:
                ge[slow].replay()
            else:
                wl.step(slow, io=io)
        b.record(cur)
        torch.cuda.synchronize()
        ems = max_over_ranks(a.elapsed_time(b))
        e2e = {"value": wl.job_tokens * K / (ems / 1e3), "unit": "tokens/s",
               "h2d_bytes_per_step": io.h2d, "d2h_bytes_per_step": io.d2h, "steps": K,
               "copies": "pinned host <-> HBM in layer groups (" + " | ".join(str(l1 - l0) for l0, l1 in io.groups) +
                         ") on a copy stream, event-ordered with compute"}

    # ---- per-kernel device time (CUDA events on the launching stream) ----
    pk = peaks()
    Lcur = wl.ctx + 1
    t_sp_iso = time_kernel(wl, "sparse", max(32, 2 * wl.L))
    t_de_iso = time_kernel(wl, "dense", max(8, wl.L // 2))
    t_de_situ, t_de_period = time_dense_in_situ(wl)
    # in situ fast step: the fast step's graph (advance + L fused launches, PDL-chained)
    # replayed back to back; its launches' average duration = step time / L
    # (the advance kernel's share is charged to them: conservative)
    t_fast_step = t_slow_step = None
    if use_graph:
        wl.set_lengths(wl.ctx + 1)
        t_fast_step = time_graph(graphs[False], 16, stream)
        wl.set_lengths(wl.ctx + 1)
        t_slow_step = time_graph(graphs[True], 3, stream)
    t_sp = t_fast_step / wl.L if t_fast_step else t_sp_iso
    t_de = t_de_situ if t_de_situ else t_de_iso
    # diagnostic: the same fused fast step with every layer in ONE launch (layer-batched
    # view of the cache), i.e. the kernel without the per-layer launch boundary
    t_lb = None
    if wl.mode in ("single", "dp"):
        try:
            lbv = wl.cache.layer_batched_view()
            qv, kv_, vv_, ov = (x.reshape(-1, *x.shape[2:]) for x in (wl.q, wl.k_new, wl.v_new, wl.out))
            s_ = torch.cuda.current_stream()
            lbv.fast_decode(0, qv, kv_, vv_, ov, prefetch=True)
            torch.cuda.synchronize()
            ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ea.record(s_)
            for _ in range(5):
                lbv.fast_decode(0, qv, kv_, vv_, ov, prefetch=True)
            eb.record(s_)
            torch.cuda.synchronize()
            t_lb = ea.elapsed_time(eb) / 5 / wl.L
            del lbv
        except Exception:
            t_lb = None
    t_sel, t_cb = time_selector(wl, max(6, wl.L // 4))
    bsp, bde, bslow = wl.bytes_sparse(), wl.bytes_dense(Lcur), wl.bytes_slow_layer(Lcur)
    hbm = pk["hbm_gbs"]
    kernels = {
        "fast_decode": {"ms": t_sp, "GB/s": bsp / t_sp / 1e6, "bytes": bsp, "isolated_ms": t_sp_iso,
                        "isolated_frac": bsp / t_sp_iso / 1e6 / hbm,
                        "layer_batched": (None if t_lb is None else
                                          {"ms_per_layer": t_lb, "GB/s": bsp / t_lb / 1e6,
                                           "frac": bsp / t_lb / 1e6 / hbm,
                                           "note": "diagnostic: all layers in one launch (no per-layer boundary)"}),
                        "timing": ("in situ: fast-step graph replay / layers (PDL chain)" if t_fast_step
                                   else "isolated launches queued back to back")},
        "dense_decode": {"ms": t_de, "GB/s": bde / t_de / 1e6, "bytes": bde,
                         "isolated_ms": t_de_iso, "isolated_frac": bde / t_de_iso / 1e6 / hbm,
                         "main_chain_period_ms": t_de_period,
                         "timing": ("in situ: the async slow step's share grid beside the Selector + compact "
                                    "(events on the main stream right before and after each dense launch, eager "
                                    "step; main_chain_period_ms adds the ring append and the logit-slot waits)"
                                    if t_de_situ else "isolated full-grid launches queued back to back")},
        "selector": {"ms": t_sel, "timing": "isolated, queued back to back"},
        "compact_build": {"ms": t_cb, "timing": "isolated, queued back to back"},
    }
    for kk in ("fast_decode", "dense_decode"):
        kernels[kk]["frac"] = kernels[kk]["GB/s"] / hbm
    share_sp = (K - n_slow) * wl.L * t_sp
    share_de = n_slow * wl.L * t_de
    dom = "fast_decode" if share_sp >= share_de else "dense_decode"
    traffic, tsrc = traffic_for(dom, cfg_name)
    roof = {"kernel": dom, "bound": "hbm", "achieved": kernels[dom]["GB/s"], "peak": hbm,
            "peak_source": pk["source"], "unit": "GB/s", "frac": kernels[dom]["frac"],
            "traffic": traffic, "traffic_source": tsrc, "algorithmic_bytes": kernels[dom]["bytes"],
            "timing": kernels[dom]["timing"], "isolated_frac": kernels[dom]["isolated_frac"],
            "share_of_step": (share_sp if dom == "fast_decode" else share_de) / ms}
    if t_slow_step:
        roof["slow_step"] = {"us": t_slow_step * 1e3, "algorithmic_bytes": wl.L * bslow,
                             "GB/s": wl.L * bslow / t_slow_step / 1e6,
                             "frac": wl.L * bslow / t_slow_step / 1e6 / hbm,
                             "note": "whole slow step (graph replay): dense KV + logits + Selector inputs "
                                     "+ compact gather r/w + appends, per layer x layers"}
    if t_fast_step:
        roof["fast_step"] = {"us": t_fast_step * 1e3, "algorithmic_bytes": wl.L * bsp,
                             "frac": wl.L * bsp / t_fast_step / 1e6 / hbm}
        fl = launch_floor_ms(wl)
        if fl:
            roof["fast_step"].update({
                "launch_floor_us_per_layer": fl * 1e3, "us_per_layer": t_sp * 1e3,
                "vs_launch_floor": t_sp / fl,
                "floor_note": "graph of 1 + L empty kernels with the fast step's PDL protocol and grid"})
    fast_us = wl.L * (t_sp * 1e3)
    res = {
        "metric": metric_name(cfg_name),
        "value": value, "unit": "tokens/s", "n_gpus": world, "steps": K, "warmup": W,
        "ms_per_step": ms / K, "higher_is_better": True,
        "scaling": "strong" if wl.mode in ("heads", "seq") else "weak", "vs_baseline": None,
        "dtype": "bf16 KV, fp32 accumulate; fp64 Selector", "data": f"synthetic ({args.inputs})",
        "config": config_dict(cfg_name, world),
        "run": {"kv_heads_per_gpu": wl.H, "batch_per_gpu": wl.B, "slow_steps_timed": f"{n_slow} of {K}",
                "cuda_graphs": use_graph if graph_note is None else graph_note,
                "slow_step": "synchronous" if wl.exec is None else
                             f"C++ DecodeExecutor: async pipeline, dense on the main stream (share grid), Selector + "
                             f"compact on an aux stream, {wl.exec.logits.shape[0]}-slot logit ring; steps "
                             f"replayed from CUDA graphs",
                "exchange": {"nccl": "ncclAllGather in-call through the C ABI (torch's communicator)",
                             "allgather": "torch.distributed all-gather",
                             "peer": "peer memory (CUDA IPC over NVLink)"}.get(wl.exchange, "none"),
                "kv_cache_gb_per_gpu": round(2 * c.sizes["kv_cache"] / 1e9, 1)},
        "slow_steps": n_slow, "fast_step_us_kernels": fast_us,
        "fast_step_us_graph": t_fast_step * 1e3 if t_fast_step else None,
        "slow_step_us_graph": t_slow_step * 1e3 if t_slow_step else None,
        "slow_step_us_kernels": wl.L * (t_de_iso + t_sel + t_cb) * 1e3,
        "kernels": kernels, "roofline": roof,
        "gpu_launches": sum(wl.launches(s_) for s_ in timed),
        "clocks": clk.summary(),
        "e2e": e2e,
    }
    if full and rank == 0 and world == 1 and not args.no_cpu:
        res["cpu_baseline"] = cpu_baseline(wl, sched[W:W + K], args)
    _release(graphs, ge)
    del wl
    _release()
    return res


def _nccl_evidence() -> dict | None:
    """NCCL's own INIT log lines of this rank (nranks, transports), when the
    bench routed NCCL_DEBUG to a file."""
    path = os.environ.get("SFI_NCCL_LOG")
    if not path:
        return None
    import glob

    lines = []
    for fn in sorted(glob.glob(path.replace("%p", "*").replace("%h", "*"))):
        try:
            with open(fn) as f:
                lines += [ln.strip() for ln in f if "nranks" in ln or "NVLS" in ln or "Init COMPLETE" in ln]
        except OSError:
            pass
    return {"log_lines": lines[:12]} if lines else None


def gpu_arm(args) -> dict:
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if world > 1:
        if args.backend == "nccl":
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            log = os.environ.setdefault("NCCL_DEBUG_FILE", f"/tmp/sfi_bench_nccl.{os.getpid()}.%h.%p.log")
            os.environ["SFI_NCCL_LOG"] = log
        dist.init_process_group(args.backend)
    if args.backend == "gloo":  # testing: several ranks may share one GPU
        local %= torch.cuda.device_count()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    red_dev = dev if args.backend == "nccl" else torch.device("cpu")

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], device=red_dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    ctx = dict(world=world, rank=rank, local=local, dev=dev, max_over_ranks=max_over_ranks)
    primary = args.config or ("c2" if world == 1 else "c3")
    if args.also is None:
        also = ["c3", "c4", "c1", "c5"] if world == 1 else ["c4", "c2"]
    else:
        also = [x for x in args.also.split(",") if x and x != "none"]
    also = [a for a in also if a != primary]
    res = run_config(primary, args, ctx, full=True)
    extra = []
    for cfg in also:
        try:
            if cfg == "c5":
                if world == 1:
                    extra.append(run_c5(dev))
                continue
            r = run_config(cfg, args, ctx, full=False)
            extra.append({k: r[k] for k in ("metric", "value", "unit", "n_gpus", "steps", "ms_per_step", "scaling",
                                            "slow_steps", "fast_step_us_graph", "slow_step_us_graph", "roofline",
                                            "config", "gpu_launches")})
        except Exception as ex:  # an extra line never costs the headline
            extra.append({"config": cfg, "error": f"{type(ex).__name__}: {ex}"[:300]})
            _release()
    res["also"] = extra
    if world > 1:
        ev = _nccl_evidence()
        res["nccl"] = {"nranks": world, "version": ".".join(map(str, torch.cuda.nccl.version())),
                       "backend": args.backend, **(ev or {})}
        dist.destroy_process_group()
    return res if rank == 0 else None


# ---------------------------------------------------------------------------
# CPU reference (oracle/_ref = the unmodified reference, else the port)

class CpuSample:
    """One layer of the workload on the reference CPU path, split into the
    independent units BASELINE.md §4 names: one reference KvStore per (request,
    KV head) (fp32, bf16-exact values; a one-head store performs exactly the
    per-head arithmetic of attend, attention.cpp:80-113, 258-291), and one
    run_selector call per request (cross-head couples a request's heads,
    selector.cpp:204-230) followed by the reorganize of its heads.
      fast unit (b, h): attention_kernel_sparse
      slow: attention_kernel_dense per (b, h), then per b run_selector on the
            workload's pooled logits + reorganize of its H stores."""

    def __init__(self, data: dict, threads: int):
        from oracle import oracle as O

        self.orc = O.load("best")
        self.kind = self.orc.kind
        self.d = data
        B, H = data["B"], data["H"]
        self.units = [(b, h) for b in range(B) for h in range(H)]
        self.cur_sel = {(b, h): data["sel"][b][h] for b, h in self.units}
        self.pool = cf.ThreadPoolExecutor(max_workers=threads)  # persistent: no per-layer thread start-up
        self.stores = dict(zip(self.units, self.pool.map(self._make_store, self.units)))

    def _make_store(self, bh):
        b, h = bh
        d = self.d
        G, D = d["Hq"] // d["H"], HEAD_DIM
        st = self.orc.store(1, 1, G, D, d["L"] + 8)
        st.append_many(d["k"][b][:, h * D:(h + 1) * D], d["v"][b][:, h * D:(h + 1) * D])
        st.reorganize(0, d["sink"], [d["sel"][b][h]])
        return st

    def _q(self, b, h):
        G, D = self.d["Hq"] // self.d["H"], HEAD_DIM
        return self.d["q"][b][h * G * D:(h + 1) * G * D]

    def fast(self, bh):
        d = self.d
        self.stores[bh].attention_sparse(0, self._q(*bh), d["sink"], [self.cur_sel[bh]], d["rs"], d["rl"])

    def dense(self, bh):
        self.stores[bh].attention_dense(0, self._q(*bh))

    def select(self, b):
        from oracle import oracle as O

        d = self.d
        sel, _ = self.orc.run_selector(d["logits"][b], np.arange(d["j0"], d["j1"] + 1), d["norms"][b],
                                       O.make_cfg(k_budget=d["K"]))
        for h in range(d["H"]):
            self.stores[(b, h)].reorganize(0, d["sink"], [sel[h]])
            self.cur_sel[(b, h)] = sel[h]


def time_cpu_layer(sample: CpuSample, slow: bool, threads: int) -> float:
    """Seconds for one layer of the workload with `threads` host threads."""
    t0 = time.perf_counter()
    if threads == 1:
        for u in sample.units:
            (sample.dense if slow else sample.fast)(u)
        if slow:
            for b in range(sample.d["B"]):
                sample.select(b)
    else:
        ex = sample.pool
        list(ex.map(sample.dense if slow else sample.fast, sample.units))
        if slow:
            list(ex.map(sample.select, range(sample.d["B"])))
    return time.perf_counter() - t0


def host_threads() -> int:
    """std::thread::hardware_concurrency() of this host (the CPUs this process may use)."""
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


def pooled_logits_np(k: np.ndarray, q: np.ndarray, H: int, Hq: int, j0: int, j1: int) -> np.ndarray:
    """The workload's mean-pooled decode logits over J (attention.cpp:394-409):
    per KV head, mean over its G query heads of q . k / sqrt(d) (input
    preparation for the Selector, untimed)."""
    G, D = Hq // H, HEAD_DIM
    kh = k.reshape(k.shape[0], H, D)[j0 - 1:j1].astype(np.float64)        # [n][H][d]
    qh = q.reshape(H, G, D)
    lg = np.einsum("nhd,hgd->hgn", kh, qh) / np.sqrt(D)
    return lg.mean(axis=1)


def gather_cpu_data(wl: Workload) -> dict:
    """Layer 0 of the running workload, read back from the device: K/V, q, the
    current selection, the pooled logits and the key norms."""
    t = wl.torch
    c = wl.cache
    t.cuda.synchronize()
    L = int(c.prefix_len[0].item())
    rl = int(c.recent_len[0].item())
    ns = int(c.n_sink_b[0].item())
    j0, j1 = ns + 1, L - rl
    # make layer 0's pooled logits current for the Selector input
    c.dense_decode(0, wl.q[0], wl.out[0], wl.logits, 0)
    t.cuda.synchronize()
    B, H, d = wl.B, wl.H, HEAD_DIM
    k = c.k_cache[0, :, :, :L].float().cpu().numpy()  # [B][H][L][d]
    v = c.v_cache[0, :, :, :L].float().cpu().numpy()
    return {
        "B": B, "H": H, "Hq": wl.Hq, "L": L, "K": wl.K, "sink": list(range(1, ns + 1)),
        "rs": L - rl + 1, "rl": rl, "j0": j0, "j1": j1,
        "k": [np.ascontiguousarray(np.transpose(k[b], (1, 0, 2)).reshape(L, H * d)) for b in range(B)],
        "v": [np.ascontiguousarray(np.transpose(v[b], (1, 0, 2)).reshape(L, H * d)) for b in range(B)],
        "q": [wl.q[0, b].double().cpu().numpy().reshape(-1) for b in range(B)],
        "sel": [[c.sel[0, b, h, : int(c.n_sel[0, b, h])].cpu().numpy() for h in range(H)] for b in range(B)],
        "logits": [wl.logits[b, :, : j1 - j0 + 1].double().cpu().numpy() for b in range(B)],
        "norms": [c.key_norms[0, b, :, j0 - 1:j1].cpu().numpy() for b in range(B)],
    }


def synth_cpu_data(cfg_name: str, inputs: str = "peaked") -> dict:
    """The workload's layer generated on the host (numpy; bf16-exact N(0,1) K/V,
    fp64 q, 32 planted k = 3 q + noise positions per (b, KV head) when peaked),
    for the reference arm: no device code involved. The Selector gets the
    workload's real pooled logits over these K and q; the first selection is the
    reference Selector's own on them."""
    name, n_layers, Hq, H, B, ctx, ns, K, R = CONFIGS[cfg_name]
    rng = np.random.default_rng(2026 + 1)
    L = ctx + 1
    rl = min(R, L - ns)
    j0, j1 = ns + 1, L - rl
    d, G = HEAD_DIM, Hq // H

    def bf16(x):
        u = np.ascontiguousarray(x, np.float32).view(np.uint32).astype(np.uint64)
        return (((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16).astype(np.uint32).view(np.float32).reshape(x.shape)

    ks, vs, norms, logits, qs = [], [], [], [], []
    for b in range(B):
        k = bf16(rng.standard_normal((L, H * d), dtype=np.float32))
        v = bf16(rng.standard_normal((L, H * d), dtype=np.float32))
        q = rng.standard_normal(Hq * d)
        if inputs == "peaked":
            kh = k.reshape(L, H, d)
            for h in range(H):
                pos = rng.integers(j0, j1 + 1, size=32)
                for i, p in enumerate(pos):
                    g = i % G
                    kh[p - 1, h] = bf16(3.0 * q[(h * G + g) * d:(h * G + g + 1) * d].astype(np.float32)
                                        + rng.standard_normal(d, dtype=np.float32))
        kh = k.reshape(L, H, d)
        norms.append(np.sqrt((kh[j0 - 1:j1].astype(np.float64) ** 2).sum(-1)).T.copy())
        logits.append(pooled_logits_np(k, q, H, Hq, j0, j1))
        ks.append(k)
        vs.append(v)
        qs.append(q)
    from oracle import oracle as O

    orc = O.load("best")
    sels = [orc.run_selector(logits[b], np.arange(j0, j1 + 1), norms[b], O.make_cfg(k_budget=K))[0]
            for b in range(B)]
    return {"B": B, "H": H, "Hq": Hq, "L": L, "K": K, "sink": list(range(1, ns + 1)),
            "rs": L - rl + 1, "rl": rl, "j0": j0, "j1": j1, "k": ks, "v": vs,
            "q": qs, "sel": sels, "logits": logits, "norms": norms, "n_layers": n_layers, "name": name,
            "ctx": ctx}


def _median(xs):
    return float(np.median(xs))


def cpu_full_step(data: dict, n_layers: int, threads: int, frac_slow: float) -> dict:
    """Un-extrapolated: every layer of one fast and one slow step actually run
    (n_layers independent per-layer store sets over the same layer inputs; the
    arithmetic does not depend on the values), on `threads` threads. Used where
    it is small enough (C1: 28 layers x 8 KV heads x 8K)."""
    samples = [CpuSample(data, threads) for _ in range(n_layers)]
    units = [(s, u) for s in samples for u in s.units]
    ex = samples[0].pool

    def run(slow):
        t0 = time.perf_counter()
        list(ex.map(lambda su: (su[0].dense if slow else su[0].fast)(su[1]), units))
        if slow:
            list(ex.map(lambda sb: sb[0].select(sb[1]), [(s, b) for s in samples for b in range(data["B"])]))
        return time.perf_counter() - t0
    run(False)
    tf = _median([run(False) for _ in range(3)])
    ts = run(True)
    step = frac_slow * ts + (1 - frac_slow) * tf
    return {"value": data["B"] / step, "unit": "tokens/s", "cores": threads, "layers": n_layers,
            "fast_step_ms": tf * 1e3, "slow_step_ms": ts * 1e3,
            "note": f"all {n_layers} layers run (no extrapolation over layers), slow fraction {frac_slow:.3f}"}


def cpu_baseline(wl: Workload, sched_timed: list[bool], args) -> dict:
    """the reference CPU path on this host, on layer 0 of the same
    workload (the device's K/V, q, selection and pooled logits), N =
    hardware_concurrency threads over (request, KV head) units, plus the
    single-thread figure; bench_attention protocol (1 discarded warm-up, median
    of repeats, harness.cpp:518-551); one layer measured, extrapolated x layers at
    the timed schedule's slow fraction."""
    data = gather_cpu_data(wl)
    N = host_threads()
    sample = CpuSample(data, N)
    time_cpu_layer(sample, False, N)  # warm-up
    tf = [time_cpu_layer(sample, False, N) for _ in range(3)]
    ts = [time_cpu_layer(sample, True, N) for _ in range(1)]
    t_fast, t_slow = _median(tf), _median(ts)
    tf1 = time_cpu_layer(sample, False, 1)
    ts1 = time_cpu_layer(sample, True, 1)
    frac_slow = sum(sched_timed) / max(1, len(sched_timed))
    step_s = wl.L * (frac_slow * t_slow + (1 - frac_slow) * t_fast)
    step_s1 = wl.L * (frac_slow * ts1 + (1 - frac_slow) * tf1)
    full = cpu_full_step(data, wl.L, N, frac_slow) if wl.cfg_name == "c1" else None
    return {"value": wl.B / step_s, "unit": "tokens/s", "cores": N, "kind": sample.kind,
            "single_thread": {"value": wl.B / step_s1, "unit": "tokens/s", "fast_layer_ms": tf1 * 1e3,
                              "slow_layer_ms": ts1 * 1e3},
            "sample": (f"layer 0 of {wl.L} measured (all {wl.B} requests x {wl.H} KV heads at L={data['L']}, "
                       f"{N} threads over {len(sample.units)} (request, KV head) units): fast "
                       f"(attention_kernel_sparse) {t_fast*1e3:.1f} ms, slow (attention_kernel_dense + "
                       f"run_selector + reorganize) {t_slow*1e3:.1f} ms per layer; extrapolated x{wl.L} layers "
                       f"at the timed schedule's slow fraction {frac_slow:.3f}"),
            "fast_layer_ms": t_fast * 1e3, "slow_layer_ms": t_slow * 1e3, "full_step_measured": full}


def reference_arm(args) -> dict | None:
    """--impl reference: the reference CPU implementation of the path (the
    unmodified reference, oracle/_ref) on this host's cores, same config / metric
    / schedule; every step is a one-layer sample of the workload (fast or slow
    per the schedule, all (request, KV head) units on hardware_concurrency
    threads) extrapolated over the layers."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return None
    cfg = args.config or ("c2" if world == 1 else "c3")
    W = args.warmup
    K = args.steps if args.steps else DEFAULT_STEPS[cfg]
    sched = schedule(W + K + 1, seed=2026 + 1)[1:]
    data = synth_cpu_data(cfg, args.inputs)
    nl = data["n_layers"]
    N = host_threads()
    sample = CpuSample(data, N)
    for i in range(W):
        time_cpu_layer(sample, sched[i], N)
    total = 0.0
    layer_s = {True: [], False: []}
    for slow in sched[W:W + K]:
        t = time_cpu_layer(sample, slow, N)
        layer_s[slow].append(t)
        total += nl * t
    B_job = data["B"] * (world if SHARDING[cfg] == "dp" else 1)
    value = B_job * K / total
    tf1 = time_cpu_layer(sample, False, 1)
    ts1 = time_cpu_layer(sample, True, 1)
    fs = sum(sched[W:W + K]) / K
    v1 = data["B"] / (nl * (fs * ts1 + (1 - fs) * tf1))
    full = cpu_full_step(data, nl, N, fs) if cfg == "c1" else None
    sample_txt = (f"each step: one layer (of {nl}) measured, all {data['B']} requests x {data['H']} KV heads "
                  f"at L={data['L']} on {N} threads over (request, KV head) units, extrapolated x{nl}; fast = "
                  "attention_kernel_sparse, slow = attention_kernel_dense + run_selector (workload's pooled "
                  "logits) + reorganize")
    return {
        "impl": "reference", "metric": metric_name(cfg),
        "value": value, "unit": "tokens/s", "n_gpus": world,
        "steps": K, "warmup": W, "ms_per_step": total / K * 1e3, "higher_is_better": True,
        "scaling": "strong" if SHARDING[cfg] in ("heads", "seq") and world > 1 else "weak",
        "vs_baseline": None, "dtype": "fp32 KV, fp64 accumulate (reference)",
        "data": f"synthetic ({args.inputs})", "config": config_dict(cfg, world),
        "measured_layer_ms": {"fast_median": _median(layer_s[False]) * 1e3 if layer_s[False] else None,
                              "slow_median": _median(layer_s[True]) * 1e3 if layer_s[True] else None},
        "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": N, "kind": sample.kind,
                         "sample": sample_txt,
                         "single_thread": {"value": v1, "unit": "tokens/s", "fast_layer_ms": tf1 * 1e3,
                                           "slow_layer_ms": ts1 * 1e3},
                         "full_step_measured": full},
        "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def spawn_ranks(args) -> int:
    """`--gpus N` without a torchrun environment: launch N ranks of this script
    through torch.distributed.run on this node (127.0.0.1) and return its exit code."""
    import socket

    import torch

    n_dev = torch.cuda.device_count()
    if args.gpus > n_dev and args.backend == "nccl":
        print(f"bench.py: --gpus {args.gpus} but only {n_dev} CUDA device(s) are visible", file=sys.stderr)
        return 2
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    import subprocess

    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None,
                    help="timed steps (default per config: C1 256, C2 512, C3/C4 64 — SURVEY §8d)")
    ap.add_argument("--warmup", type=int, default=8)
    ap.add_argument("--config", default=None, choices=sorted(CONFIGS),
                    help="headline workload (default: c2 on 1 GPU, c3 KV-head sharded on N > 1)")
    ap.add_argument("--also", default=None,
                    help="comma-separated extra configs timed after the headline (default: c3,c4,c1,c5 on 1 GPU, "
                         "c4,c2 on N > 1; 'none' for none); reported under 'also'")
    ap.add_argument("--inputs", default="peaked", choices=["peaked", "iid"],
                    help="synthetic inputs: peaked = 32 planted k = 3q + noise positions per (b, KV head) "
                         "(SURVEY §8d), iid = N(0, 1) K/V")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline leg")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--layers", type=int, default=0, help="override the layer count (testing only)")
    ap.add_argument("--sync-slow", action="store_true",
                    help="slow steps without the asynchronous Selector pipeline (one stream)")
    ap.add_argument("--backend", default=os.environ.get("SFI_DIST_BACKEND", "nccl"),
                    help="torch.distributed backend (gloo: several ranks on one GPU, testing only)")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args))
    res = reference_arm(args) if args.impl == "reference" else gpu_arm(args)
    if res is not None:
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()

"""C5 (BASELINE configs[4]): long-CoT generation on Qwen3-8B attention shapes —
2K prefill + 32K generated tokens — sweeping the refresh budget t_max and the
selected-memory size K against full-KV dense decode (every step dense over the
whole cache, no Selector).

Per K, the fast step (one fused launch per layer) and the slow step (dense +
Selector + compact, asynchronous pipeline) are timed as CUDA-graph replays at
contexts spanning the generation; a (K, t_max) schedule's time per token is
(1 - f) fast + f slow with f the slow fraction of the seeded 32K-step schedule
(triggers Bernoulli(1/24), forced at t_max; scheduler.cpp:93-99), averaged over
the generation (trapezoid over the context points). Synthetic bf16 KV, batch 8.

    python scripts/sweep_c5.py [--batch 8] [--out profiles/r02/c5_sweep.json]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2603_12038_b200 as sfi  # noqa: E402

L, HQ, H, D, NS, R = 36, 32, 8, 128, 4, 256
PREFILL, GEN = 2048, 32768
CTX = [PREFILL, PREFILL + GEN // 4, PREFILL + GEN // 2, PREFILL + 3 * GEN // 4, PREFILL + GEN]
KS = [512, 1024, 2048, 3836]
TMAX = [16, 32, 64, 128]


def slow_fraction(t_max: int, steps: int = GEN, seed: int = 2031) -> float:
    rng = np.random.default_rng(seed)
    since, trig, n = 0, True, 0
    for _ in range(steps):
        slow = trig or since + 1 >= t_max
        n += slow
        since = 0 if slow else since + 1
        trig = bool(rng.random() < bench.P_TRIGGER)
    return n / steps


def graph(fn):
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    return g


def replay_ms(g, reps):
    return bench.time_graph(g, reps, torch.cuda.current_stream())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=8)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02", "c5_sweep.json"))
    args = ap.parse_args()
    B = args.batch
    dev = torch.device("cuda", 0)
    Lmax = CTX[-1] + 64
    g0 = torch.Generator().manual_seed(2031)
    q = torch.randn(L, B, HQ, D, generator=g0).to(dev)
    kn = torch.randn(L, B, H, D, generator=g0).to(dev).bfloat16()
    out = torch.zeros(L, B, HQ, D, device=dev)
    prm = sfi.SelectorParams()
    res = {"fast_ms": {}, "slow_ms": {}, "dense_ms": {}}
    for K in KS + [None]:  # None: the full-KV dense baseline
        c = sfi.SfiCache(L, B, H, HQ, D, Lmax, NS, K or 512, R, device=dev)
        c.fill_synthetic(seed=2031, length=CTX[-1])
        pipe = sfi.SlowStepPipeline(c)

        def fast():
            c.step_advance()
            for l in range(L):
                c.fast_decode(l, q[l], kn[l], kn[l], out[l], prefetch=True)

        def slow(rebuild=False):
            c.step_advance()
            pipe.begin()
            for l in range(L):
                pipe.layer(l, q[l], out[l], kn[l], kn[l], prm, rebuild_ring=rebuild)
            pipe.end()

        def dense():  # full-KV decode: append + dense attention over the whole cache, every step
            c.step_advance()
            for l in range(L):
                c.ring_append(l, kn[l], kn[l])
                c.dense_decode(l, q[l], out[l])

        for ctx in CTX:
            c.set_lengths([ctx] * B, [NS] * B)
            if K is None:
                gd = graph(dense)
                c.set_lengths([ctx] * B, [NS] * B)
                res["dense_ms"][ctx] = replay_ms(gd, 4)
                continue
            slow(rebuild=True)  # selection + compact cache for this context
            torch.cuda.synchronize()
            c.set_lengths([ctx] * B, [NS] * B)
            gf, gs = graph(fast), graph(slow)
            c.set_lengths([ctx] * B, [NS] * B)
            res["fast_ms"].setdefault(K, {})[ctx] = replay_ms(gf, 8)
            c.set_lengths([ctx] * B, [NS] * B)
            res["slow_ms"].setdefault(K, {})[ctx] = replay_ms(gs, 3)
            c.check_errors()
        del c, pipe
        torch.cuda.empty_cache()

    def gen_avg(per_ctx):  # mean time per step over a generation uniform in context
        ys = [per_ctx[x] for x in CTX]
        return float(np.trapezoid(ys, CTX) / (CTX[-1] - CTX[0]))

    dense_avg = gen_avg(res["dense_ms"])
    rows = []
    for K in KS:
        for t in TMAX:
            f = slow_fraction(t)
            per = {x: (1 - f) * res["fast_ms"][K][x] + f * res["slow_ms"][K][x] for x in CTX}
            avg = gen_avg(per)
            rows.append({"k_budget": K, "t_max": t, "slow_fraction": round(f, 4),
                         "tokens_per_s": B / (avg / 1e3), "dense_tokens_per_s": B / (dense_avg / 1e3),
                         "speedup_vs_full_kv": dense_avg / avg,
                         "ms_per_step_at_34k": per[CTX[-1]]})
    doc = {"workload": f"C5: Qwen3-8B-shaped attention (32 q / 8 kv heads, d 128, {L} layers), batch {B}, "
                       f"{PREFILL} prefill + {GEN} generated tokens, sink {NS}, recent {R}",
           "data": "synthetic bf16 KV (device fill), random q", "contexts": CTX,
           "timing": "CUDA-graph replays per step (CUDA events); schedule mixes by the seeded slow fraction",
           "fast_ms": {str(k): v for k, v in res["fast_ms"].items()},
           "slow_ms": {str(k): v for k, v in res["slow_ms"].items()},
           "dense_ms": res["dense_ms"], "sweep": rows}
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as fh:
        json.dump(doc, fh, indent=1)
    print(f"full-KV dense decode: {B / (dense_avg / 1e3):.0f} tokens/s")
    print("K     t_max  slow%   tokens/s  speedup")
    for r in rows:
        print(f"{r['k_budget']:<5d} {r['t_max']:<6d} {100 * r['slow_fraction']:5.2f}  {r['tokens_per_s']:8.0f}  "
              f"{r['speedup_vs_full_kv']:6.2f}x")


if __name__ == "__main__":
    main()

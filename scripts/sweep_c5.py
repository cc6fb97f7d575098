"""C5 (BASELINE configs[4]): long-CoT generation on Qwen3-8B attention shapes —
2K prefill + 32K generated tokens — sweeping the refresh budget t_max and the
selected-memory size K against full-KV dense decode (every step dense over the
whole cache, no Selector), at batch 8 and batch 1.

Per (K, batch) this is bench.run_c5: the C++ executor's fast and slow steps and
a full-KV dense step replayed from CUDA graphs at five context points of the
generation, mixed by each t_max's seeded slow fraction (triggers Bernoulli(1/24),
forced at t_max; scheduler.cpp:93-99) and averaged over the generation.

    python scripts/sweep_c5.py [--batches 8,1] [--out gpurun_out/c5_sweep.json]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402

KS = [512, 1024, 2048, 3836]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batches", default="8,1")
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "c5_sweep.json"))
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    rows, runs = [], []
    for B in [int(x) for x in args.batches.split(",")]:
        dense = None
        for i, K in enumerate(KS):
            r = bench.run_c5(dev, k_budget=K, batch=B, dense=(i == 0))
            runs.append(r)
            if i == 0:  # the first K's run of this batch times the full-KV dense step
                dense = r["full_kv_dense_tokens_per_s"]
            for s in r["sweep"]:
                rows.append({"batch": B, "k_budget": K, "t_max": s["t_max"], "slow_fraction": s["slow_fraction"],
                             "tokens_per_s": s["tokens_per_s"], "full_kv_dense_tokens_per_s": dense,
                             "speedup_vs_full_kv": s["tokens_per_s"] / dense})
    doc = {"workload": "C5: Qwen3-8B-shaped attention (32 q / 8 kv heads, d 128, 36 layers), 2048 prefill + 32768 "
                       "generated tokens, sink 4, recent 256",
           "data": "synthetic bf16 KV (device fill), random q", "timing": runs[0]["timing"],
           "sweep": rows, "runs": [{k: r[k] for k in ("config", "per_context_ms")} for r in runs]}
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as fh:
        json.dump(doc, fh, indent=1)
    print("B  K     t_max  slow%   tokens/s  full-KV   speedup")
    for r in rows:
        print(f"{r['batch']:<2d} {r['k_budget']:<5d} {r['t_max']:<6d} {100 * r['slow_fraction']:5.2f}  "
              f"{r['tokens_per_s']:8.0f}  {r['full_kv_dense_tokens_per_s']:7.0f}  {r['speedup_vs_full_kv']:6.2f}x")


if __name__ == "__main__":
    main()

"""Per-kernel microbenchmark on the C2 shapes (tuning aid, not the bench).

    SFI_DECODE_TRACE=1 [SFI_DECODE_CTAS=n] python scripts/microbench_decode.py [--layers 4]

Times sparse decode, dense decode, the three Selector kernels and compact build
with CUDA events, and (with SFI_DECODE_TRACE) prints the per-CTA timeline of
the last sparse / dense launch: prologue, first-tile latency, busy time.
"""
import argparse
import ctypes as C
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2603_12038_b200 as sfi  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--layers", type=int, default=4)
ap.add_argument("--batch", type=int, default=8)
ap.add_argument("--ctx", type=int, default=32768)
ap.add_argument("--hq", type=int, default=32)
ap.add_argument("--iters", type=int, default=20)
args = ap.parse_args()

L, B, H, Hq, d = args.layers, args.batch, 8, args.hq, 128
ctx = args.ctx
c = sfi.SfiCache(L, B, H, Hq, d, ctx + 64, 4, 2048, 256)
c.fill_synthetic(7, ctx)
c.set_lengths([ctx] * B, [4] * B)
c.step_advance()
q = torch.randn(L, B, Hq, d, device="cuda")
out = torch.zeros_like(q)
logits = c.pooled_logits
prm = sfi.SelectorParams()
for l in range(L):
    c.dense_decode(l, q[l], out[l], logits, 0)
    c.selector(l, logits, prm)
    c.compact_build(l, True)
torch.cuda.synchronize()
c.check_errors()
lib = C.CDLL(sfi.LIBRARY_PATH)


def timeit(fn, iters):
    s = torch.cuda.current_stream()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(iters)]
    for i in range(iters):
        ev[i][0].record(s)
        fn(i)
        ev[i][1].record(s)
    torch.cuda.synchronize()
    ts = [a.elapsed_time(b) * 1e3 for a, b in ev][2:]
    return float(np.median(ts)), float(np.min(ts))


def trace(tag):
    if not os.environ.get("SFI_DECODE_TRACE"):
        return
    buf = (C.c_int64 * (16 * 1024))()
    n = lib.sfi_debug_decode_trace(buf, 1024)
    a = np.frombuffer(buf, dtype=np.int64)[: 16 * n].reshape(n, 16).astype(np.float64)
    live = a[a[:, 0] > 0]
    t0 = live[:, 0].min()
    start, pro, first, end = (live[:, i] - t0 for i in range(4))
    busy = end - start
    print(f"[{tag}] ctas={n} live={len(live)} launch spread={start.max()/1e3:.2f}us "
          f"prologue med={np.median(pro-start)/1e3:.2f}us first-tile med={np.median(first-pro)/1e3:.2f}us "
          f"busy med={np.median(busy)/1e3:.2f} max={busy.max()/1e3:.2f} min={busy.min()/1e3:.2f}us "
          f"kernel span={end.max()/1e3:.2f}us emissions mean={live[:,4].mean():.2f} tiles mean={live[:,5].mean():.1f}")
    cons_end = live[:, 12] - t0
    print(f"   consumers done med={np.median(cons_end - start)/1e3:.2f}us max={cons_end.max()/1e3:.2f}us; "
          f"epilogue busy mean={live[:,7].mean():.0f}ns max={live[:,7].max():.0f}; "
          f"consumer EMPTY stall mean={live[:,8].mean():.0f}; partial+fence+atomic mean={live[:,9].mean():.0f} "
          f"max={live[:,9].max():.0f}; merge mean={live[:,10].mean():.0f} max={live[:,10].max():.0f}")
    e_first, e_last = live[:, 13] - t0, live[:, 14] - t0
    print(f"   first emission at med={np.median(e_first - start)/1e3:.2f}us, last at med={np.median(e_last - start)/1e3:.2f}us; "
          f"fence mean={live[:,9].mean():.0f} max={live[:,9].max():.0f}ns")
    slow = np.argsort(-end)[:5]
    for i in slow:
        print(f"   slow cta: start={start[i]/1e3:.2f} pro={pro[i]/1e3:.2f} first={first[i]/1e3:.2f} "
              f"end={end[i]/1e3:.2f} emis={live[i,4]:.0f} tiles={live[i,5]:.0f} sm={live[i,6]:.0f} "
              f"cons_end={cons_end[i]/1e3:.2f} epi={live[i,7]/1e3:.2f} stall={live[i,8]/1e3:.2f} "
              f"fence={live[i,9]/1e3:.2f} merge={live[i,10]/1e3:.2f}us")


def trace_fast(tag):
    if not os.environ.get("SFI_DECODE_TRACE"):
        return
    buf = (C.c_int64 * (16 * 1024))()
    n = lib.sfi_debug_decode_trace(buf, 1024)
    a = np.frombuffer(buf, dtype=np.int64)[: 16 * n].reshape(n, 16).astype(np.float64)
    live = a[a[:, 0] > 0]
    t0 = live[:, 0].min()
    rel = lambda i: (live[:, i] - t0) / 1e3
    st, wt, ft, cd, c1, md, en = rel(0), rel(1), rel(2), rel(12), rel(13), rel(14), rel(3)
    q = lambda x: f"{np.percentile(x, 10):.2f}/{np.median(x):.2f}/{x.max():.2f}"
    print(f"[{tag}] ctas={n} (p10/med/max us from first CTA start) start={q(st)} post-wait={q(wt)} "
          f"first-tile={q(ft)} consumers-done={q(cd)} cluster-sync1={q(c1)} merge-done={q(md)} end={q(en)} "
          f"tiles mean={live[:,5].mean():.1f}")
    aux = (live[:, 8] - t0) / 1e3
    aux = aux[live[:, 8] > 0]
    print(f"   consumer-loop-done={q(rel(9))} producer-issued={q(rel(10))} aux-ready(rank0)={q(aux) if len(aux) else '-'}")
    sms = live[:, 6].astype(int)
    cnt = np.bincount(sms, minlength=148)
    print(f"   CTAs per SM: {np.bincount(cnt)} ; busy(end-start) med={np.median(en-st):.2f}")


res = {}
res["sparse_us"] = timeit(lambda i: c.sparse_decode(i % L, q[i % L], out[i % L]), args.iters)
trace("sparse")
kn = torch.randn(L, B, H, d, device="cuda").bfloat16()
res["fast_us"] = timeit(lambda i: c.fast_decode(i % L, q[i % L], kn[i % L], kn[i % L], out[i % L], prefetch=True), args.iters)
trace_fast("fast single")
res["fast_noprefetch_us"] = timeit(lambda i: c.fast_decode(i % L, q[i % L], kn[i % L], kn[i % L], out[i % L]), args.iters)


def back_to_back(fn, n):  # n launches between two events (PDL overlap between launches)
    s = torch.cuda.current_stream()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for i in range(3):
        fn(i)
    a.record(s)
    for i in range(n):
        fn(i)
    b.record(s)
    torch.cuda.synchronize()
    return a.elapsed_time(b) * 1e3 / n


res["fast_b2b_us"] = back_to_back(lambda i: c.fast_decode(i % L, q[i % L], kn[i % L], kn[i % L], out[i % L], prefetch=True), 64)
trace_fast("fast b2b prefetch")
res["fast_b2b_noprefetch_us"] = back_to_back(lambda i: c.fast_decode(i % L, q[i % L], kn[i % L], kn[i % L], out[i % L]), 64)
res["sparse_b2b_us"] = back_to_back(lambda i: c.sparse_decode(i % L, q[i % L], out[i % L]), 64)
res["dense_us"] = timeit(lambda i: c.dense_decode(i % L, q[i % L], out[i % L], logits, 0), max(6, args.iters // 3))
trace("dense")
res["selector_us"] = timeit(lambda i: c.selector(i % L, logits, prm), 10)
res["compact_us"] = timeit(lambda i: c.compact_build(i % L, False), 10)
k = torch.randn(B, H, d, device="cuda").bfloat16()
res["ring_append_us"] = timeit(lambda i: c.ring_append(i % L, k, k), 10)
S = 256 + 4 + 2048
sp_bytes = B * H * S * 4 * d
de_bytes = B * H * (ctx + 1) * 4 * d
res["sparse_GBs"] = sp_bytes / res["sparse_us"][0] / 1e3
res["fast_b2b_GBs"] = sp_bytes / res["fast_b2b_us"] / 1e3
res["dense_GBs"] = de_bytes / res["dense_us"][0] / 1e3
print(json.dumps(res))
c.check_errors()


def graph_per_launch(fn, n, reps=5):
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for i in range(n):
            fn(i)
    g.replay()
    torch.cuda.synchronize()
    s = torch.cuda.current_stream()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(reps):
        g.replay()
    b.record(s)
    torch.cuda.synchronize()
    return a.elapsed_time(b) * 1e3 / (n * reps)


if not os.environ.get("SFI_DECODE_TRACE"):
    gr = {}
    gr["graph_fast_prefetch_us"] = graph_per_launch(
        lambda i: c.fast_decode(i % L, q[i % L], kn[i % L], kn[i % L], out[i % L], prefetch=True), L)
    def with_adv(i):
        if i == 0:
            c.step_advance()
        c.fast_decode(i % L, q[i % L], kn[i % L], kn[i % L], out[i % L], prefetch=True)

    gr["graph_adv_fast_prefetch_us"] = graph_per_launch(with_adv, L)
    gr["graph_fast_us"] = graph_per_launch(
        lambda i: c.fast_decode(i % L, q[i % L], kn[i % L], kn[i % L], out[i % L]), 36)
    gr["graph_sparse_us"] = graph_per_launch(lambda i: c.sparse_decode(i % L, q[i % L], out[i % L]), 36)
    gr["graph_dense_us"] = graph_per_launch(lambda i: c.dense_decode(i % L, q[i % L], out[i % L], logits, 0), 8)
    gr["graph_fast_GBs"] = sp_bytes / gr["graph_fast_prefetch_us"] / 1e3
    print(json.dumps(gr))

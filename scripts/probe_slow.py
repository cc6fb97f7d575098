"""Probe: slow-step graph time, synchronous vs asynchronous pipeline; dense variants."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench

res = {"ctas": os.environ.get("SFI_DECODE_CTAS")}
wl = bench.Workload("c2", 200, torch.device("cuda", 0))
c = wl.cache
def cap(fn):
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    return g
pipe = wl.pipe
wl.pipe = None
g_sync = cap(lambda: wl.step(True))
wl.pipe = pipe
g_async = cap(lambda: wl.step(True))
import paper_2603_12038_b200 as sfi
wl.pipe = sfi.SlowStepPipeline(c, share_sm=False)
g_async2 = cap(lambda: wl.step(True))
def dense_only(share):
    def f():
        for l in range(wl.L):
            c.dense_decode_ex(l, wl.q[l], wl.out[l], wl.logits, 0, share_sm=share)
    return f
g_d2 = cap(dense_only(False))
g_d1 = cap(dense_only(True))
def sel_only():
    for l in range(wl.L):
        c.selector(l, wl.logits, wl.params)
        c.compact_build(l)
g_sel = cap(sel_only)
for name, g in [("slow_sync", g_sync), ("slow_async", g_async), ("dense_2cta", g_d2), ("dense_1cta", g_d1), ("sel_compact", g_sel), ("slow_sync2", g_sync), ("slow_async2", g_async), ("slow_async_2cta", g_async2)]:
    wl.set_lengths(wl.ctx + 1)
    res[name + "_us_per_layer"] = bench.time_graph(g, 3) * 1e3 / wl.L
print(json.dumps(res))

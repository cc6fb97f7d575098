"""Probe: async slow step per layer with the aux-stream work trimmed (what the
Selector and the compact build cost beside the dense decode), and aux priority."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2603_12038_b200 as sfi

wl = bench.Workload("c2", 200, torch.device("cuda", 0))
c = wl.cache
res = {}


def cap(fn):
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    return g


orig_sel, orig_cb = c.selector, c.compact_build
variants = {
    "both": (orig_sel, orig_cb),
    "no_aux": (lambda *a, **k: None, lambda *a, **k: None),
    "compact_only": (lambda *a, **k: None, orig_cb),
    "selector_only": (orig_sel, lambda *a, **k: None),
}
for share in (True, False):
    for name, (fs, fc) in variants.items():
        c.selector, c.compact_build = fs, fc
        wl.pipe = sfi.SlowStepPipeline(c, share_sm=share)
        g = cap(lambda: wl.step(True))
        wl.set_lengths(wl.ctx + 1)
        res[f"{name}_share{int(share)}"] = bench.time_graph(g, 3) * 1e3 / wl.L
c.selector, c.compact_build = orig_sel, orig_cb
# high-priority aux stream
p = sfi.SlowStepPipeline(c, share_sm=True)
p.aux = torch.cuda.Stream(device=c.k_cache.device, priority=-1)
wl.pipe = p
g = cap(lambda: wl.step(True))
wl.set_lengths(wl.ctx + 1)
res["both_share1_auxhi"] = bench.time_graph(g, 3) * 1e3 / wl.L
print(json.dumps({k: round(v, 1) for k, v in res.items()}))

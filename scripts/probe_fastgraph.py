"""Probe: fast-step graph time inside the bench workload vs variants."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench

wl = bench.Workload("c2", 200, torch.device("cuda", 0))
c = wl.cache
res = {}
def cap(fn):
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    return g
g_step = cap(lambda: wl.step(False))
def only_fast():
    for l in range(wl.L):
        c.fast_decode(l, wl.q[l], wl.k_new[l], wl.v_new[l], wl.out[l], prefetch=True)
g_fast = cap(only_fast)
def fast_same_inputs():
    for l in range(wl.L):
        c.fast_decode(l, wl.q[0], wl.k_new[0], wl.v_new[0], wl.out[0], prefetch=True)
g_same = cap(fast_same_inputs)
for name, g in [("step", g_step), ("only_fast", g_fast), ("same_inputs", g_same), ("step2", g_step)]:
    c.set_lengths([wl.ctx + 1] * wl.B, [wl.ns] * wl.B)
    res[name] = bench.time_graph(g, 16) * 1e3 / wl.L
print(json.dumps(res))

"""Probe: C4 fast-step graph time per layer (run once per SFI_FAST_CLUSTER value)."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench

cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
wl = bench.Workload(cfg, 200, torch.device("cuda", 0))
c = wl.cache
res = {"cluster_env": os.environ.get("SFI_FAST_CLUSTER", "auto")}


def cap(fn):
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    return g


for pf in (True, False):
    def only_fast(pf=pf):
        for l in range(wl.L):
            c.fast_decode(l, wl.q[l], wl.k_new[l], wl.v_new[l], wl.out[l], prefetch=pf)
    g = cap(only_fast)
    c.set_lengths([wl.ctx + 1] * wl.B, [wl.ns] * wl.B)
    res[f"graph_us_per_layer_prefetch{int(pf)}"] = bench.time_graph(g, 16) * 1e3 / wl.L
# one isolated launch (stream, no graph)
st = torch.cuda.current_stream()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ts = []
for i in range(20):
    c.set_lengths([wl.ctx + 1] * wl.B, [wl.ns] * wl.B)
    torch.cuda.synchronize()
    e0.record(st)
    c.fast_decode(0, wl.q[0], wl.k_new[0], wl.v_new[0], wl.out[0], prefetch=False)
    e1.record(st)
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1) * 1e3)
res["isolated_us_median"] = sorted(ts)[len(ts) // 2]
print(json.dumps(res))

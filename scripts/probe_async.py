"""Probe: which aux-stream work bounds the asynchronous slow step (us per layer)."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench

wl = bench.Workload("c2", 200, torch.device("cuda", 0))
c = wl.cache
pipe = wl.pipe
main = None
aux = pipe.aux

def slow(kind):
    def f():
        global main
        main = torch.cuda.current_stream()
        aux.wait_stream(main)
        c.step_advance()
        for l in range(wl.L):
            s = l % pipe.slots
            if l >= pipe.slots:
                main.wait_event(pipe.ev_free[s])
            if kind != "noappend":
                c.ring_append(l, wl.k_new[l], wl.v_new[l])
            c.dense_decode_ex(l, wl.q[l], wl.out[l], pipe.logits[s], 0, share_sm=True)
            pipe.ev_ready[s].record(main)
            with torch.cuda.stream(aux):
                aux.wait_event(pipe.ev_ready[s])
                if kind in ("sel", "all"):
                    c.selector(l, pipe.logits[s], wl.params)
                if kind in ("compact", "all"):
                    c.compact_build(l)
                pipe.ev_free[s].record(aux)
        main.wait_stream(aux)
    return f

res = {}
graphs = {}
for kind in ("noappend", "none", "sel", "compact", "all"):
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        slow(kind)()
    graphs[kind] = g
for kind, g in graphs.items():
    wl.set_lengths(wl.ctx + 1)
    res[kind] = bench.time_graph(g, 3) * 1e3 / wl.L
print(json.dumps(res))

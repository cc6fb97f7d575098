"""Probe: per-layer timeline of one asynchronous slow step (C2): CUDA events after
each layer's dense decode (main stream) and after its Selector + compact build
(aux stream) — shows which chain the slow step waits on."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2603_12038_b200 as sfi  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
wl = bench.Workload(cfg, 200, torch.device("cuda", 0))
c = wl.cache
pipe = sfi.SlowStepPipeline(c)
ev_d = [torch.cuda.Event(enable_timing=True) for _ in range(wl.L)]
ev_a = [torch.cuda.Event(enable_timing=True) for _ in range(wl.L)]
start = torch.cuda.Event(enable_timing=True)


def run():
    wl.set_lengths(wl.ctx + 1)
    torch.cuda.synchronize()
    start.record()
    pipe.begin()
    for l in range(wl.L):
        pipe.layer(l, wl.q[l], wl.out[l], wl.k_new[l], wl.v_new[l], wl.params, False)
        ev_d[l].record(pipe.main)
        ev_a[l].record(pipe.aux)
    pipe.end()
    torch.cuda.synchronize()


for _ in range(3):
    run()
d = [start.elapsed_time(e) * 1e3 for e in ev_d]
a = [start.elapsed_time(e) * 1e3 for e in ev_a]
print(json.dumps({"dense_done_us": [round(x, 1) for x in d], "aux_done_us": [round(x, 1) for x in a],
                  "aux_lag_us": [round(y - x, 1) for x, y in zip(d, a)]}))

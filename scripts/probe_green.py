"""Probe: async slow step with the Selector + compact chain confined to an SM
partition (CUDA green context) so the dense decode keeps its own SMs."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2603_12038_b200 as sfi  # noqa: E402
from cuda.bindings import driver as cu  # noqa: E402


def chk(r):
    err = r[0] if isinstance(r, tuple) else r
    if err != cu.CUresult.CUDA_SUCCESS:
        raise RuntimeError(str(err))
    return r[1:] if isinstance(r, tuple) and len(r) > 1 else None


def _ctx_stream(dev, res):
    (desc,) = chk(cu.cuDevResourceGenerateDesc([res], 1))
    (g,) = chk(cu.cuGreenCtxCreate(desc, dev, cu.CUgreenCtxCreate_flags.CU_GREEN_CTX_DEFAULT_STREAM))
    (st,) = chk(cu.cuGreenCtxStreamCreate(g, cu.CUstream_flags.CU_STREAM_NON_BLOCKING, 0))
    return g, st


def green_streams(n_sms: int):
    """(aux stream on n_sms SMs, dense stream on the remaining SMs)."""
    torch.cuda.init()
    (dev,) = chk(cu.cuDeviceGet(torch.cuda.current_device()))
    (res,) = chk(cu.cuDeviceGetDevResource(dev, cu.CUdevResourceType.CU_DEV_RESOURCE_TYPE_SM))
    groups, n_groups, rem = chk(cu.cuDevSmResourceSplitByCount(1, res, 0, n_sms))
    g0 = groups[0] if isinstance(groups, (list, tuple)) else groups
    ga, sa = _ctx_stream(dev, g0)
    gd, sd = _ctx_stream(dev, rem)
    return (ga, gd), sa, sd


res = {}
wl = bench.Workload("c2", 200, torch.device("cuda", 0))
c = wl.cache


def cap(fn):
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    return g


for share in (True, False):
    wl.pipe = sfi.SlowStepPipeline(c, share_sm=share)
    g = cap(lambda: wl.step(True))
    wl.set_lengths(wl.ctx + 1)
    res[f"default_share{int(share)}"] = bench.time_graph(g, 3) * 1e3 / wl.L
for n in (40, 52, 64):
    try:
        ctxs, sa, sd = green_streams(n)
        for share in (True, False):
            p = sfi.SlowStepPipeline(c, share_sm=share)
            p.aux = torch.cuda.ExternalStream(int(sa))
            wl.pipe = p
            dense_stream = torch.cuda.ExternalStream(int(sd))
            with torch.cuda.stream(dense_stream):
                for _ in range(2):
                    wl.set_lengths(wl.ctx + 1)
                    wl.step(True)
                torch.cuda.synchronize()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                wl.set_lengths(wl.ctx + 1)
                a.record(dense_stream)
                for _ in range(3):
                    wl.step(True)
                b.record(dense_stream)
            torch.cuda.synchronize()
            res[f"green{n}_share{int(share)}_eager"] = a.elapsed_time(b) / 3 * 1e3 / wl.L
    except Exception as e:  # noqa: BLE001
        res[f"green{n}"] = repr(e)[:300]
# eager reference for the default path
wl.pipe = sfi.SlowStepPipeline(c, share_sm=True)
for _ in range(2):
    wl.step(True)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(3):
    wl.step(True)
b.record()
torch.cuda.synchronize()
res["default_share1_eager"] = a.elapsed_time(b) / 3 * 1e3 / wl.L
c.check_errors()
print(json.dumps({k: (round(v, 1) if isinstance(v, float) else v) for k, v in res.items()}))

"""Probe: timeline of one graph-replayed fast step, per layer (SFI_LAYER_TRACE=1)."""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2603_12038_b200 as sfi  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
wl = bench.Workload(cfg, 200, torch.device("cuda", 0), sync_slow=True)  # per-layer launches from Python
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    wl.step(False)
for _ in range(3):
    wl.set_lengths(wl.ctx + 1)
    g.replay()
    torch.cuda.synchronize()
lib = C.CDLL(sfi.LIBRARY_PATH)
L, M = wl.L, 1024
buf = (C.c_int64 * (L * M * 16))()
n = lib.sfi_debug_layer_trace(buf, L, M)
a = np.frombuffer(buf, dtype=np.int64).reshape(L, M, 16)[:, :n].astype(np.float64)
t0 = a[0, :, 0].min()
rows = []
for l in range(L):
    x = a[l]
    st, wt, ft, en = x[:, 0] - t0, x[:, 1] - t0, x[:, 2] - t0, x[:, 3] - t0
    rows.append((st.min(), np.median(st), st.max(), wt.min(), np.median(wt), ft.min(), np.median(ft), np.median(en), en.max()))
print("layer: start(min/med/max) post-wait(min/med) first-tile(min/med) end(med/max)   [us from layer-0 first start]")
for l, r in enumerate(rows):
    r = [v / 1e3 for v in r]
    gap = (rows[l][0] - rows[l - 1][8]) / 1e3 if l else 0.0
    print(f"{l:2d}: {r[0]:7.2f} {r[1]:7.2f} {r[2]:7.2f} | {r[3]:7.2f} {r[4]:7.2f} | {r[5]:7.2f} {r[6]:7.2f} | {r[7]:7.2f} {r[8]:7.2f}  "
          f"span={r[8]-r[0]:5.2f} start-after-prev-end={gap:6.2f} postwait-after-prev-end={(rows[l][3]-rows[l-1][8])/1e3 if l else 0:6.2f}")
print("per-layer period (first start to first start):", np.diff([r[0] for r in rows]).mean() / 1e3, "us")

# phase medians within a layer, relative to that CTA's own start:
# 10 producer pre-wait TMA issued, 1 griddep wait returned, 2 first tile landed,
# 9 consumer loop done, 12 ring-drained barrier, 11 partials written, 15 CTA combine,
# 13 cluster sync, 14 merge, 3 end
idx = [10, 1, 2, 9, 12, 11, 15, 13, 14, 3]
ph = np.stack([np.median(a[l][:, idx] - a[l][:, :1], axis=0) for l in range(1, L)]).mean(0) / 1e3
print("phase medians (us after CTA start), idx", idx, ":", np.round(ph, 2).tolist())
os.makedirs("gpurun_out", exist_ok=True)
np.save(f"gpurun_out/layer_trace_{cfg}.npy", a)
cyc = np.stack([np.median(a[l][:, [4, 7]], axis=0) for l in range(1, L)]).mean(0)
print("median cycles: receive wait, merge:", cyc.tolist())

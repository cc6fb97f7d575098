"""Probe: the asynchronous slow step's two chains, per layer, from the executor's
hook events (one eager slow step): main stream — dense launch duration and the
gap before it (logit-slot wait + ring append); aux stream — the Selector and
the compact rebuild, and how far the aux chain lags the main chain.

    python scripts/probe_pipeline.py [c2|c3|c4]   (env as for bench.py)
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
wl = bench.Workload(cfg, 64, torch.device("cuda", 0))
L = wl.L
mk = lambda: [torch.cuda.Event(enable_timing=True) for _ in range(L)]  # noqa: E731
res = []
for rep in range(3):
    bd, ad, ab, asel, ae = mk(), mk(), mk(), mk(), mk()
    t0 = torch.cuda.Event(enable_timing=True)
    for e in bd + ad + ab + asel + ae:
        e.record()
    wl.set_lengths(wl.ctx)
    torch.cuda.synchronize()
    t0.record(wl.exec.stream)
    wl.exec.step(True, wl.q, wl.k_new, wl.v_new, wl.out, False, (), ad, origin=wl.exec.stream,
                 record_before_attention=bd, aux_events=(ab, asel, ae))
    torch.cuda.synchronize()
    T = lambda e: t0.elapsed_time(e) * 1e3  # noqa: E731  us since the step's start
    rows = [{"dense_start": T(bd[l]), "dense_end": T(ad[l]), "sel_start": T(ab[l]), "sel_end": T(asel[l]),
             "compact_end": T(ae[l])} for l in range(L)]
    res.append(rows)
rows = res[-1]
mid = range(2, L - 1)
out = {
    "config": cfg, "layers": L,
    "dense_us": float(np.mean([r["dense_end"] - r["dense_start"] for r in (rows[l] for l in mid)])),
    "main_gap_us": float(np.mean([rows[l]["dense_start"] - rows[l - 1]["dense_end"] for l in mid])),
    "selector_us": float(np.mean([r["sel_end"] - r["sel_start"] for r in (rows[l] for l in mid)])),
    "compact_us": float(np.mean([r["compact_end"] - r["sel_end"] for r in (rows[l] for l in mid)])),
    "aux_gap_us": float(np.mean([rows[l]["sel_start"] - rows[l - 1]["compact_end"] for l in mid])),
    "aux_lag_us": float(np.mean([r["compact_end"] - r["dense_end"] for r in (rows[l] for l in mid)])),
    "last_dense_end_us": rows[-1]["dense_end"], "last_compact_end_us": rows[-1]["compact_end"],
}
print(json.dumps(out))
for l in (0, 1, 2, L // 2, L - 2, L - 1):
    r = rows[l]
    print(f"layer {l:3d}: dense {r['dense_start']:9.1f} -> {r['dense_end']:9.1f} | selector {r['sel_start']:9.1f} -> "
          f"{r['sel_end']:9.1f} | compact -> {r['compact_end']:9.1f}")

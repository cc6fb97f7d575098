"""Per-CTA timeline of one dense decode (SFI_DECODE_TRACE=1): mma.sync vs tcgen05."""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_12038_b200 as sfi  # noqa: E402
from paper_2603_12038_b200 import SfiCache  # noqa: E402

lib = C.CDLL(sfi.LIBRARY_PATH)
cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
B, H, Hq, L = {"c2": (8, 8, 32, 32768), "c3": (4, 8, 64, 131072), "c4": (1, 4, 64, 262144)}[cfg]
c = SfiCache(1, B, H, Hq, 128, L + 8, 4, 64, 32)
c.fill_synthetic(seed=3, length=L)
c.set_lengths([L] * B, [4] * B)
q = torch.randn(B, Hq, 128).cuda()
out = torch.zeros_like(q)
lg = torch.zeros_like(c.pooled_logits)
for k in ("mma", "tc"):
    for _ in range(3):
        c.dense_decode_ex(0, q, out, lg, 0, kernel=k)
    torch.cuda.synchronize()
    buf = (C.c_int64 * (16 * 1024))()
    n = lib.sfi_debug_decode_trace(buf, 1024)
    a = np.frombuffer(buf, dtype=np.int64)[: 16 * n].reshape(n, 16).astype(np.float64)
    live = a[a[:, 0] > 0]
    t0 = live[:, 0].min()
    st, pro, first, end = (live[:, i] - t0 for i in range(4))
    loop_end = live[:, 12] - t0
    print(f"[{cfg} {k}] ctas={n} start spread {st.max()/1e3:.1f}us prologue med {np.median(pro-st)/1e3:.2f} "
          f"first tile med {np.median(first-pro)/1e3:.2f} loop end med {np.median(loop_end)/1e3:.1f} "
          f"max {loop_end.max()/1e3:.1f} | end med {np.median(end)/1e3:.1f} max {end.max()/1e3:.1f}us "
          f"merge max {live[:,10].max()/1e3:.1f}us tiles {live[:,5].min():.0f}-{live[:,5].max():.0f}")

"""One dense decode at a BASELINE config through the tcgen05 kernel (for ncu)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_12038_b200 import SfiCache  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
kernel = sys.argv[2] if len(sys.argv) > 2 else "tc"
B, H, Hq, L = {"c2": (8, 8, 32, 32768), "c3": (4, 8, 64, 131072), "c4": (1, 4, 64, 262144)}[cfg]
c = SfiCache(1, B, H, Hq, 128, L + 8, 4, 64, 32)
c.fill_synthetic(seed=3, length=L)
c.set_lengths([L] * B, [4] * B)
q = torch.randn(B, Hq, 128).cuda()
out = torch.zeros_like(q)
lg = torch.zeros_like(c.pooled_logits)
for _ in range(3):
    c.dense_decode_ex(0, q, out, lg, 0, kernel=kernel)
torch.cuda.synchronize()
print("ok")

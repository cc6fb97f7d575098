"""Generates tests/golden/reference_vectors.json by running the UNMODIFIED
reference (oracle/_ref/libsfi_ref.so, built from /root/reference/proj/src by
oracle/Makefile) on small seeded inputs. Run here (where /root/reference
exists); the JSON is committed and travels to the GPU box.

    python tests/golden/make_golden.py
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from helpers import bf16_round  # noqa: E402
from oracle import oracle as O  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "reference_vectors.json")


def selector_cases(ref):
    cases = []
    rng = np.random.default_rng(2026)
    specs = [
        dict(H=1, n=2, W=1, cfg={}),
        dict(H=2, n=9, W=1, cfg=dict(k_budget=3)),
        dict(H=3, n=50, W=1, cfg=dict(k_budget=8)),
        dict(H=3, n=50, W=4, cfg=dict(k_budget=8, alpha=0.5)),
        dict(H=4, n=120, W=1, cfg=dict(k_budget=20, gamma=0.5, beta=2.0, p_curve=1.5, eta=0.0,
                                       lambda_clip=0.5, alpha_soft=0.3, alpha_cross=0.7,
                                       temperature=0.5, nms_radius=1)),
        dict(H=8, n=300, W=1, cfg=dict(k_budget=40, pool=1)),
        dict(H=2, n=30, W=1, cfg=dict(k_budget=100)),
        dict(H=2, n=30, W=1, cfg=dict(k_budget=0)),
    ]
    for i, sp in enumerate(specs):
        H, n, W = sp["H"], sp["n"], sp["W"]
        allowed = (np.cumsum(rng.integers(1, 4, size=n)) + 4).astype(np.int32)
        vals = np.round(rng.normal(0, 1.5, size=(H, W * n)), 6)
        norms = np.round(np.abs(rng.normal(8, 2, size=(H, n))) + 0.1, 6)
        cfg = O.make_cfg(**sp["cfg"])
        sel, st = ref.run_selector(vals, allowed, norms, cfg, width=W, stages=True)
        cases.append(dict(name=f"selector_{i}", H=H, n=n, W=W, cfg=sp["cfg"],
                          allowed=allowed.tolist(), values=vals.tolist(), norms=norms.tolist(),
                          selected=[s.tolist() for s in sel],
                          z_adj=st["z_adj"].tolist(), lambda_star=st["lambda"].tolist()))
    return cases


def topk_cases(ref):
    rng = np.random.default_rng(6)
    cases = []
    for t in range(40):
        n = int(rng.integers(1, 13))
        k = int(rng.integers(0, 7))
        pos = (np.cumsum(rng.integers(1, 5, size=n))).astype(np.int32)
        sc = rng.uniform(-1, 1, size=n)
        if t % 2 == 0:
            sc = np.round(sc * 4) / 4
        cases.append(dict(scores=sc.tolist(), positions=pos.tolist(), k=k,
                          want=ref.select_top_k(sc, pos, k).tolist()))
    return cases


def attention_cases(ref):
    rng = np.random.default_rng(31)
    cases = []
    for (H, Hq, d, L) in [(2, 4, 16, 40), (2, 8, 128, 97), (1, 1, 64, 33)]:
        k = bf16_round(rng.normal(size=(L, H * d)))
        v = bf16_round(rng.normal(size=(L, H * d)))
        st = ref.store(1, H, Hq, d, 4096)
        st.append_many(k, v)
        q = rng.normal(size=Hq * d)
        dense, reads = st.attention_dense(0, q)
        ns = min(4, L)
        rl = 8
        sink = list(range(1, ns + 1))
        sel = [sorted(rng.choice(np.arange(ns + 1, L - rl + 1), size=6, replace=False).tolist())
               for _ in range(H)]
        st.reorganize(0, sink, sel)
        sparse, sreads = st.attention_sparse(0, q, sink, sel, L - rl + 1, rl)
        compact = [st.compact(0, h)[0].tolist() for h in range(H)]
        norms = [[st.key_norm(0, h, p) for p in range(1, L + 1)] for h in range(H)]
        cases.append(dict(H=H, Hq=Hq, d=d, L=L, k=k.tolist(), v=v.tolist(), q=q.tolist(),
                          dense=dense.tolist(), dense_reads=reads, sink=sink, selected=sel,
                          recent_start=L - rl + 1, recent_len=rl, sparse=sparse.tolist(),
                          sparse_reads=sreads, compact_positions=compact, key_norms=norms))
    return cases


def main():
    O.build(ref=True)
    ref = O.load("reference")
    assert ref.kind == "reference"
    data = dict(
        generator="tests/golden/make_golden.py",
        source="/root/reference/proj/src (unmodified) via oracle/_ref/libsfi_ref.so",
        selector=selector_cases(ref),
        top_k=topk_cases(ref),
        attention=attention_cases(ref),
        recent_window=[dict(prefix=p, n_sink=4, n_recent=8, want=list(ref.recent_window(p, 4, 8)))
                       for p in (1, 2, 4, 6, 12, 40)],
    )
    with open(OUT, "w") as f:
        json.dump(data, f, separators=(",", ":"))
    print("wrote", OUT, os.path.getsize(OUT), "bytes")


if __name__ == "__main__":
    main()

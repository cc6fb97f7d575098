"""CPU: the oracle is pinned before it is trusted.

* the C restatement (oracle/liboracle.so) reproduces the golden vectors that
  the unmodified reference produced (tests/golden/reference_vectors.json,
  made by tests/golden/make_golden.py) bit for bit;
* it reproduces the reference's own known-answer tests
  (proj/tests/test_selector.cpp, test_oracle.cpp, test_scheduler.cpp);
* where the reference library is built here (oracle/_ref), port == reference
  bitwise on fresh seeded inputs, stage arrays included.
"""
from __future__ import annotations

import itertools
import json
import math
import os

import numpy as np
import pytest

from helpers import bf16_round
from oracle import oracle as O

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "reference_vectors.json")


@pytest.fixture(scope="module")
def gold():
    with open(GOLD) as f:
        return json.load(f)


@pytest.fixture(scope="module")
def port():
    return O.load("port")


def test_port_matches_golden_selector(gold, port):
    for case in gold["selector"]:
        cfg = O.make_cfg(**case["cfg"])
        sel, st = port.run_selector(np.array(case["values"]), np.array(case["allowed"]),
                                    np.array(case["norms"]), cfg, width=case["W"], stages=True)
        for h in range(case["H"]):
            assert sel[h].tolist() == case["selected"][h], case["name"]
        assert np.array_equal(st["z_adj"], np.array(case["z_adj"])), case["name"]
        assert st["lambda"].tolist() == case["lambda_star"], case["name"]


def test_port_matches_golden_top_k(gold, port):
    for case in gold["top_k"]:
        got = port.select_top_k(np.array(case["scores"]), np.array(case["positions"]), case["k"])
        assert got.tolist() == case["want"]


def test_port_matches_golden_attention(gold, port):
    for case in gold["attention"]:
        st = port.store(1, case["H"], case["Hq"], case["d"], 4096)
        st.append_many(np.array(case["k"], np.float32), np.array(case["v"], np.float32))
        q = np.array(case["q"])
        dense, reads = st.attention_dense(0, q)
        assert np.array_equal(dense, np.array(case["dense"])) and reads == case["dense_reads"]
        st.reorganize(0, case["sink"], case["selected"])
        for h in range(case["H"]):
            assert st.compact(0, h)[0].tolist() == case["compact_positions"][h]
            assert [st.key_norm(0, h, p) for p in range(1, case["L"] + 1)] == case["key_norms"][h]
        sparse, sreads = st.attention_sparse(0, q, case["sink"], case["selected"],
                                             case["recent_start"], case["recent_len"])
        assert np.array_equal(sparse, np.array(case["sparse"])) and sreads == case["sparse_reads"]


def test_port_matches_golden_recent_window(gold, port):
    for case in gold["recent_window"]:
        assert list(port.recent_window(case["prefix"], case["n_sink"], case["n_recent"])) == case["want"]


# ---- reference known-answer tests (proj/tests/*.cpp) ------------------------

def test_evidence_w1_is_softmax(port):  # test_selector.cpp:52-60
    _, st = port.run_selector([[0.0, math.log(2.0)]], [5, 9], [[1.0, 1.0]], stages=True)
    assert st["evidence"][0] == pytest.approx([1 / 3, 2 / 3], rel=1e-12)


def test_evidence_symmetric_one_hot_alpha_half(port):  # test_selector.cpp:62-73
    _, st = port.run_selector([[0.0, -1e30, -1e30, 0.0]], [3, 4], [[1.0, 1.0]],
                              O.make_cfg(alpha=0.5), width=2, stages=True)
    assert st["evidence"][0] == pytest.approx([0.5, 0.5], rel=1e-12)


def test_evidence_alpha_one_is_row_mean(port):  # test_selector.cpp:75-88
    v = [math.log(0.8), math.log(0.2), math.log(0.4), math.log(0.6)]
    _, st = port.run_selector([v], [1, 2], [[1.0, 1.0]], width=2, stages=True)
    mu0, mu1 = 0.6, 0.4
    assert st["evidence"][0] == pytest.approx([mu0 / (mu0 + mu1), mu1 / (mu0 + mu1)], rel=1e-12)


def test_prior_key_norm_downweighting(port):  # test_selector.cpp:140-150
    _, st = port.run_selector([[0.0, 0.0]], [1, 2], [[1.0, 3.0]],
                              O.make_cfg(gamma=1.0, beta=0.0, eta=0.0), stages=True)
    assert st["prior"][0] == pytest.approx([0.75, 0.25], rel=1e-6)


def test_prior_position_decay(port):  # test_selector.cpp:119-138
    allowed = [10, 20, 30, 40, 50]
    _, st = port.run_selector([[0.0] * 5], allowed, [[1.0] * 5],
                              O.make_cfg(gamma=0.0, beta=1.0, p_curve=1.0, eta=0.0), stages=True)
    e = [math.exp(-(a - 10) / (40 + 1e-8)) for a in allowed]
    assert st["prior"][0] == pytest.approx([x / sum(e) for x in e], rel=1e-12)


def test_fuse_saturates_clip(port):  # test_selector.cpp:160-170
    f = [0.5, 0.3, 0.2]
    _, st = port.run_selector([[math.log(x) for x in f]], [1, 2, 3], [[2.0] * 3],
                              O.make_cfg(beta=0.0, eta=0.0), stages=True)
    assert st["lambda"][0] == pytest.approx(0.02, rel=1e-12)
    s = np.exp(st["z_base"][0]) - 1e-8
    assert s == pytest.approx([0.4966666666666667, 0.3006666666666667, 0.2026666666666667], rel=1e-9)


def test_soft_nms_examples(port):  # test_selector.cpp:217-229
    z = [1.0, 0.5, 0.2]
    assert port.refine_soft_nms(z, O.make_cfg(alpha_soft=0.0, nms_radius=1)).tolist() == z
    assert port.refine_soft_nms(z, O.make_cfg(alpha_soft=0.5, nms_radius=1)) == pytest.approx([1.0, 0.25, 0.05])


def test_cross_head_examples(port):  # test_selector.cpp:261-280
    one = [[0.3, -1.0, 2.0]]
    assert port.refine_cross_head(one).tolist() == one
    two = [[0.3, 1.0], [0.1, 1.0]]
    assert port.refine_cross_head(two, O.make_cfg(alpha_cross=0.0)).tolist() == two
    out = port.refine_cross_head([[1.0], [1.0]])
    assert out[:, 0] == pytest.approx([1.0 + 0.35 * math.log(0.5)] * 2, rel=1e-12)


def test_select_top_k_examples(port):  # test_selector.cpp:295-301
    assert port.select_top_k([0.1, 0.9, 0.5, 0.9], [10, 20, 30, 40], 2).tolist() == [20, 40]
    assert port.select_top_k([0.9, 0.5, 0.5], [10, 20, 30], 2).tolist() == [10, 20]
    assert port.select_top_k([0.9, 0.5], [10, 20], 0).tolist() == []
    assert port.select_top_k([0.1, 0.2], [10, 20], 5).tolist() == [10, 20]
    with pytest.raises(O.OracleError) as e:
        port.select_top_k([0.1], [1], -1)
    assert e.value.name == "out_of_range"


def _exhaustive_top_k(scores, positions, k):
    """oracle.cpp:164-199: max-sum k-subset, ties -> lexicographically smallest."""
    n = len(scores)
    if k >= n:
        return list(positions)
    if k <= 0:
        return []
    best, best_sum = None, -math.inf
    for idx in itertools.combinations(range(n), k):
        s = sum(scores[i] for i in idx)
        t = [positions[i] for i in idx]
        if s > best_sum or (s == best_sum and t < best):
            best, best_sum = t, s
    return best


def test_top_k_matches_exhaustive_with_ties(port):  # oracle.cpp:540-562
    rng = np.random.default_rng(16)
    for trial in range(300):
        n = int(rng.integers(1, 11))
        k = int(rng.integers(0, 7))
        pos = np.cumsum(rng.integers(1, 5, size=n)).tolist()
        sc = rng.uniform(-1, 1, size=n)
        if rng.random() < 0.5:
            sc = np.round(sc * 4) / 4
        assert port.select_top_k(sc, pos, k).tolist() == _exhaustive_top_k(sc.tolist(), pos, k)


def test_run_selector_refinements_off_is_top_k_of_evidence(port):  # test_selector.cpp:303-325
    rng = np.random.default_rng(5)
    n = 24
    allowed = [5 + 2 * i for i in range(n)]
    vals = rng.normal(0, 2, size=(1, n))
    cfg = O.make_cfg(alpha_soft=0.0, alpha_cross=0.0, lambda_clip=0.0, k_budget=4)
    sel, st = port.run_selector(vals, allowed, [[1.0] * n], cfg, stages=True)
    assert sel[0].tolist() == port.select_top_k(st["evidence"][0], allowed, 4).tolist()


def test_recent_window_rule(port):  # test_scheduler.cpp:178-191
    for prefix in (2, 4, 6, 12, 40):
        rs, rl = port.recent_window(prefix, 4, 8)
        assert rl == max(0, min(8, prefix - min(4, prefix)))
        if rl:
            assert rs + rl - 1 == prefix


def test_error_paths(port):
    with pytest.raises(O.OracleError) as e:
        port.run_selector([[0.0, float("nan")]], [1, 2], [[1.0, 1.0]])
    assert e.value.name == "non_finite_input"
    with pytest.raises(O.OracleError) as e:
        port.run_selector([[0.0, 1.0]], [1, 2], [[1.0, -1.0]])
    assert e.value.name == "non_finite_input"
    st = port.store(1, 2, 4, 16, 64)
    rng = np.random.default_rng(0)
    st.append_many(bf16_round(rng.normal(size=(30, 32))), bf16_round(rng.normal(size=(30, 32))))
    with pytest.raises(O.OracleError) as e:
        st.reorganize(0, [1, 2, 3], [[3], []])
    assert e.value.name == "overlap_violation"
    with pytest.raises(O.OracleError) as e:
        st.reorganize(0, [1, 2, 3], [[500], []])
    assert e.value.name == "out_of_range"
    st.reorganize(0, [1, 2], [[7], [7]])
    with pytest.raises(O.OracleError) as e:
        st.attention_sparse(0, np.ones(64), [1, 2], [[8], [7]], 26, 5)
    assert e.value.name == "stale_compact"


# ---- port == reference bitwise on fresh inputs (when built here) -------------

needs_ref = pytest.mark.skipif(not O.have_reference(), reason="oracle/_ref not built (no /root/reference)")


@needs_ref
def test_port_equals_reference_selector_random():
    ref, port = O.load("reference"), O.load("port")
    rng = np.random.default_rng(123)
    for trial in range(25):
        H = int(rng.integers(1, 9))
        n = int(rng.integers(1, 4000))
        W = int(rng.choice([1, 1, 1, 3, 16]))
        allowed = np.cumsum(rng.integers(1, 3, size=n)).astype(np.int32) + 4
        vals = rng.normal(0, 1, size=(H, W * n)).astype(np.float32).astype(np.float64)
        norms = np.abs(rng.normal(8, 2, size=(H, n)))
        cfg = O.make_cfg(k_budget=int(rng.integers(0, 600)), alpha=float(rng.choice([1.0, 0.5, 0.3])))
        a, sa = ref.run_selector(vals, allowed, norms, cfg, width=W, stages=True)
        b, sb = port.run_selector(vals, allowed, norms, cfg, width=W, stages=True)
        assert all(np.array_equal(x, y) for x, y in zip(a, b)), trial
        for key in sa:
            assert np.array_equal(sa[key], sb[key]), (trial, key)


@needs_ref
def test_port_equals_reference_attention_random():
    ref, port = O.load("reference"), O.load("port")
    rng = np.random.default_rng(7)
    for (H, Hq, d, L) in [(2, 4, 16, 200), (8, 32, 128, 300), (4, 64, 128, 150)]:
        k = bf16_round(rng.normal(size=(L, H * d)))
        v = bf16_round(rng.normal(size=(L, H * d)))
        stores = [o.store(1, H, Hq, d, 4096) for o in (ref, port)]
        for st in stores:
            st.append_many(k, v)
        q = rng.normal(size=Hq * d)
        a, b = (st.attention_dense(0, q) for st in stores)
        assert np.array_equal(a[0], b[0]) and a[1] == b[1]
        sel = [sorted(rng.choice(np.arange(5, L - 16), size=20, replace=False).tolist()) for _ in range(H)]
        for st in stores:
            st.reorganize(0, [1, 2, 3, 4], sel)
        a, b = (st.attention_sparse(0, q, [1, 2, 3, 4], sel, L - 15, 16) for st in stores)
        assert np.array_equal(a[0], b[0]) and a[1] == b[1]
        for h in range(H):
            pa, ka, va = stores[0].compact(0, h)
            pb, kb, vb = stores[1].compact(0, h)
            assert np.array_equal(pa, pb) and np.array_equal(ka, kb) and np.array_equal(va, vb)
            assert stores[0].key_norm(0, h, 17) == stores[1].key_norm(0, h, 17)


@needs_ref
@pytest.mark.parametrize("pool", [0, 1])
def test_port_capture_equals_reference_run_step(pool):
    """Pins the port's slow-step logit capture (orc_dense_capture, the oracle the
    GPU pooled logits are checked against) to the reference's own run_step
    capture (attention.cpp:367-409) on a toy-model step: the reference hands back
    the window it captured, the attention context, the paged K/V and the query;
    the port, given that K/V and query, reproduces window and context."""
    ref, port = O.load("reference"), O.load("port")
    spec = dict(n_layers=2, n_query_heads=8, n_kv_heads=2, head_dim=32, vocab_size=64, max_positions=256)
    rng = np.random.default_rng(40 + pool)
    tokens = rng.integers(5, 64, size=90)
    allowed = np.arange(5, 90 - 16 + 1)          # J = [n_sink + 1, L - recent], contiguous in decode
    r = ref.toy_capture(spec, 17, tokens, allowed, pool)
    st = port.store(1, spec["n_kv_heads"], spec["n_query_heads"], spec["head_dim"], 256)
    st.append_many(r["k"], r["v"])
    out, lg = st.dense_capture(0, r["q"], allowed, pool)
    assert np.abs(out - r["context"]).max() <= 1e-12 * np.abs(r["context"]).max()
    assert np.abs(lg - r["logits"]).max() <= 1e-12 * np.abs(r["logits"]).max()
    assert np.array_equal(lg, r["logits"]) and np.array_equal(out, r["context"])  # bit-identical in practice

"""The reference's Selector stage API on the device (selector.hpp:84-122,
module.cpp:80-143): evidence_from_window, prior_from_stats, fuse,
refine_soft_nms, refine_cross_head, normalize and run_selector with a
SelectorTrace, each checked stage by stage against the unmodified reference's
SelectorTrace arrays (oracle/_ref: z_base, z_nms, z_adj, evidence, prior,
lambda*) on identical inputs.

Bar: the stage arrays within 1e-12 (relative to the row's largest magnitude —
tree-ordered fp64 sums and CUDA's exp/log/pow vs glibc differ by ulps), lambda*
within 1e-12, the selections bit-exact; error codes as the reference's.
"""
from __future__ import annotations

import math

import numpy as np
import pytest

from helpers import oracle

pytestmark = pytest.mark.gpu

TOL = 1e-12


def _sfi():
    import paper_2603_12038_b200 as sfi

    return sfi


def _close(got, want, tol=TOL):
    got, want = np.asarray(got, np.float64), np.asarray(want, np.float64)
    scale = max(np.abs(want).max(), 1e-300)
    return np.abs(got - want).max() <= tol * scale


def _case(rng, H, n, W, masked):
    allowed = (np.cumsum(rng.integers(1, 3, size=n)) + 4).astype(np.int32)
    vals = rng.normal(0.0, 1.2, size=(H, W * n))
    if masked:
        m = rng.random((H, W * n)) < 0.15
        m[:, :n] = False  # keep row 0 live
        vals[m] = -1e30
    norms = np.abs(rng.normal(9.0, 2.5, size=(H, n))) + 0.05
    return allowed, vals, norms


CASES = [
    # H, n, W, masked, config overrides
    (1, 2, 1, False, {}),
    (4, 700, 1, False, {}),
    (8, 3000, 1, False, dict(alpha_cross=0.0)),
    (3, 400, 16, True, dict(alpha=0.5)),
    (2, 1500, 4, True, dict(alpha=0.3, gamma=0.7, beta=2.0, p_curve=1.5, eta=0.25, lambda_clip=0.4,
                            alpha_soft=0.8, alpha_cross=0.1, temperature=0.7, nms_radius=3)),
]


@pytest.mark.parametrize("H,n,W,masked,kw", CASES)
def test_stage_arrays_match_reference_trace(H, n, W, masked, kw):
    sfi = _sfi()
    from oracle import oracle as O

    rng = np.random.default_rng(H * 100 + n + W)
    allowed, vals, norms = _case(rng, H, n, W, masked)
    K = max(1, n // 5)
    cfg = sfi.SelectorConfig()
    for k, v in dict(kw, k_budget=K).items():
        setattr(cfg, k, v)
    want_sel, ref = oracle("reference").run_selector(vals, allowed, norms, O.make_cfg(k_budget=K, **kw),
                                                     width=W, stages=True)
    w = sfi.LogitWindow()
    w.width, w.allowed, w.values = W, allowed.tolist(), vals.tolist()
    stats = sfi.make_cache_stats(norms.tolist(), allowed.tolist(), cfg.epsilon)
    # the stage functions one by one
    f = sfi.evidence_from_window(w, cfg)
    r = sfi.prior_from_stats(stats, allowed.tolist(), cfg)
    assert len(f) == H and len(r) == H
    for h in range(H):
        assert list(f[h].support) == allowed.tolist() and sfi.validate_distribution(f[h])
        assert _close(f[h].mass, ref["evidence"][h]), ("evidence", h)
        assert _close(r[h].mass, ref["prior"][h]), ("prior", h)
        fs = sfi.fuse(f[h], r[h], cfg)
        assert abs(fs.lambda_star - ref["lambda"][h]) <= TOL, ("lambda", h)
        z = [math.log(m + cfg.epsilon) for m in fs.fused.mass]  # the check only; the device forms z in run_selector
        assert _close(z, ref["z_base"][h], 1e-11), ("z_base via fuse", h)
        nms = sfi.refine_soft_nms(ref["z_base"][h].tolist(), cfg)
        assert _close(nms, ref["z_nms"][h]), ("soft_nms", h)
    cross = sfi.refine_cross_head(ref["z_nms"].tolist(), cfg)
    assert _close(cross, ref["z_adj"]), "cross_head"
    # run_selector with a trace: the staged device pipeline end to end
    tr = sfi.SelectorTrace()
    tr.capture_stages = True
    sel = sfi.run_selector(w, stats, cfg, tr)
    for h in range(H):
        assert np.array_equal(np.asarray(sel[h], np.int32), want_sel[h]), ("selection", h)
        assert _close(tr.stages.base[h], ref["z_base"][h])
        assert _close(tr.stages.after_nms[h], ref["z_nms"][h])
        assert _close(tr.stages.after_cross[h], ref["z_adj"][h])
        assert abs(tr.fusion[h].lambda_star - ref["lambda"][h]) <= TOL
    # and without stages: the fused device Selector, same selections
    plain = sfi.run_selector(w, stats, cfg)
    assert all(np.array_equal(np.asarray(a, np.int32), b) for a, b in zip(plain, want_sel))


def test_stage_known_answers():
    """test_selector.cpp KATs through the stage functions."""
    sfi = _sfi()
    cfg = sfi.SelectorConfig()
    w = sfi.LogitWindow()
    w.width, w.allowed, w.values = 1, [5, 9], [[0.0, math.log(2.0)]]
    f = sfi.evidence_from_window(w, cfg)[0]
    assert f.mass == pytest.approx([1 / 3, 2 / 3], rel=1e-12)
    fs = sfi.fuse(sfi.ScoreDistribution([1, 2, 3], [0.5, 0.3, 0.2]),
                  sfi.ScoreDistribution([1, 2, 3], [1 / 3, 1 / 3, 1 / 3]), cfg)
    assert fs.lambda_star == 0.02
    assert fs.fused.mass == pytest.approx([0.4966666666666667, 0.3006666666666667, 0.2026666666666667], rel=1e-14)
    r1 = sfi.SelectorConfig()
    r1.nms_radius = 1
    assert sfi.refine_soft_nms([1.0, 0.5, 0.2], r1) == pytest.approx([1.0, 0.25, 0.05], rel=1e-15)
    assert sfi.refine_cross_head([[1.0], [1.0]], cfg)[0][0] == pytest.approx(1 + 0.35 * math.log(0.5), rel=1e-15)
    d = sfi.normalize([1, 2, 4], [1.0, 1.0, 2.0])
    assert list(d.support) == [1, 2, 4] and d.mass == [0.25, 0.25, 0.5]


def test_stage_error_codes():
    """distribution.cpp:41-60 / selector.cpp:54-160 error paths."""
    sfi = _sfi()
    cfg = sfi.SelectorConfig()

    def code(fn):
        with pytest.raises(sfi.SfiError) as e:
            fn()
        return e.value.code

    assert code(lambda: sfi.normalize([], [])) == "empty_support"
    assert code(lambda: sfi.normalize([1, 2], [1.0])) == "support_mismatch"
    assert code(lambda: sfi.normalize([1, 2], [1.0, -1.0])) == "non_finite_input"
    assert code(lambda: sfi.normalize([1, 2], [0.0, 0.0])) == "empty_support"
    w = sfi.LogitWindow()
    w.width, w.allowed, w.values = 1, [1, 2], [[0.0, float("inf")]]
    assert code(lambda: sfi.evidence_from_window(w, cfg)) == "non_finite_input"
    w.values = [[-1e30, -1e30]]
    assert code(lambda: sfi.evidence_from_window(w, cfg)) == "empty_support"
    w.values = [[0.0, 1.0], [0.0]]
    assert code(lambda: sfi.evidence_from_window(w, cfg)) == "support_mismatch"
    w.width = 0
    assert code(lambda: sfi.evidence_from_window(w, cfg)) == "out_of_range"
    st = sfi.make_cache_stats([[1.0, float("nan")]], [1, 2], 1e-8)
    assert code(lambda: sfi.prior_from_stats(st, [1, 2], cfg)) == "non_finite_input"
    assert code(lambda: sfi.prior_from_stats(st, [1, 2, 3], cfg)) == "support_mismatch"
    assert code(lambda: sfi.fuse(sfi.ScoreDistribution([1], [1.0]), sfi.ScoreDistribution([2], [1.0]), cfg)) == \
        "support_mismatch"
    assert code(lambda: sfi.refine_cross_head([[1.0, 2.0], [1.0]], cfg)) == "support_mismatch"
    assert sfi.refine_cross_head([], cfg) == []

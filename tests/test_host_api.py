"""CPU: the host-side half of the reference-facing API (configs, CacheStats,
scheduler bookkeeping) reproduces the reference's known answers
(proj/tests/test_core.cpp, test_scheduler.cpp, python/test_smoke.py)."""
from __future__ import annotations

import pytest

import paper_2603_12038_b200 as sfi


def test_default_config_values():  # test_core.cpp:20-44, test_smoke.py:11-22
    cfg = sfi.default_config()
    assert cfg.limits.n_sink == 4 and cfg.limits.n_recent == 256 and cfg.limits.k_budget == 2048
    assert cfg.selector.k_budget == 2048
    assert cfg.trigger.t_max == 64 and cfg.trigger.window_decode == 1
    assert cfg.trigger.window_prefill == 16
    s = cfg.selector
    assert (s.lambda_clip, s.alpha_soft, s.alpha_cross, s.epsilon) == (0.02, 0.5, 0.35, 1e-8)
    assert (s.alpha, s.gamma, s.beta, s.p_curve, s.eta, s.temperature, s.nms_radius) == \
        (1.0, 1.0, 1.0, 2.0, 0.5, 1.0, 2)
    assert cfg.trigger.trigger_tokens == [0, 1, 2, 3, 4]
    cfg.validate()


def test_config_validation():
    s = sfi.SelectorConfig()
    s.alpha = 0.0
    with pytest.raises(sfi.SfiError) as e:
        s.validate()
    assert e.value.code == "config"


def test_cache_stats():  # test_selector.cpp:100-107, 152-158
    st = sfi.make_cache_stats([[1.0, 1.0, 1.0]], [10, 20, 70], 1e-8)
    assert (st.j_min, st.j_max) == (10, 70)
    assert st.normalized_pos[0] == 0.0
    assert st.normalized_pos[-1] == pytest.approx(1.0, rel=1e-8)
    with pytest.raises(sfi.SfiError) as e:
        sfi.make_cache_stats([[1.0, 1.0]], [1, 2, 3], 1e-8)
    assert e.value.code == "support_mismatch"
    with pytest.raises(sfi.SfiError) as e:
        sfi.make_cache_stats([], [], 1e-8)
    assert e.value.code == "empty_support"


def test_compute_allowed_examples():  # test_scheduler.cpp:68-83
    s = sfi.SparseState()
    s.sink, s.recent_start, s.recent_len = [1], 8, 3
    assert sfi.compute_allowed(s, 10) == [2, 3, 4, 5, 6, 7]
    s2 = sfi.SparseState()
    s2.sink, s2.recent_start, s2.recent_len = [1, 2], 3, 4
    assert sfi.compute_allowed(s2, 6) == []
    assert sfi.compute_allowed(sfi.SparseState(), 4) == [1, 2, 3, 4]


def test_trigger_policy():  # test_scheduler.cpp:85-100
    lim = sfi.CacheLimits()
    lim.n_sink, lim.n_recent = 2, 4
    trig = sfi.TriggerConfig()
    trig.trigger_tokens = [9]
    st = sfi.init_decode_state(16, 1, 1, lim)
    st.t, st.last_token = 1, 9
    assert sfi.next_step_type(st, trig) == 1
    st.last_token, st.steps_since_slow = 5, 3
    assert sfi.next_step_type(st, trig) == 0


def test_t_max_forces_slow_on_64th_step():  # test_scheduler.cpp:102-124
    lim = sfi.CacheLimits()
    lim.n_sink, lim.n_recent = 1, 4
    trig = sfi.TriggerConfig()
    trig.trigger_tokens = [9]
    st = sfi.init_decode_state(8, 1, 1, lim)
    st.last_token = 1
    first = -1
    for step in range(1, 71):
        if sfi.next_step_type(st, trig) == 1:
            first = step
            assert st.steps_since_slow == 63
            sfi.slow_step_update(st, [[[]]], lim)
            assert st.steps_since_slow == 0
            break
        sfi.fast_step_update(st, lim)
    assert first == 64


def test_fast_and_slow_updates():  # test_scheduler.cpp:126-176
    lim = sfi.CacheLimits()
    lim.n_sink, lim.n_recent, lim.k_budget = 2, 4, 8
    st = sfi.init_decode_state(20, 2, 2, lim)
    pl = st.per_layer
    pl[0].selected = [[5, 9], [6]]
    st.per_layer = pl
    before = st.per_layer[0].recent_start
    sfi.fast_step_update(st, lim)
    assert st.per_layer[0].selected == [[5, 9], [6]]
    assert st.per_layer[0].recent_start == before + 1 and st.per_layer[0].recent_len == 4
    assert (st.t, st.prefix_len, st.steps_since_slow) == (1, 21, 1)
    lim.k_budget = 4
    st = sfi.init_decode_state(20, 1, 1, lim)
    st.steps_since_slow = 17
    sfi.slow_step_update(st, [[[3, 11]]], lim)
    assert st.per_layer[0].selected == [[3, 11]] and st.steps_since_slow == 0
    for bad in ([[[1]]], [[[20]]], [[[5, 6, 7, 8, 9]]]):
        st = sfi.init_decode_state(20, 1, 1, lim)
        with pytest.raises(sfi.SfiError) as e:
            sfi.slow_step_update(st, bad, lim)
        assert e.value.code in ("overlap_violation", "out_of_range")


def test_recent_window_rule():  # test_scheduler.cpp:178-191
    lim = sfi.CacheLimits()
    lim.n_sink, lim.n_recent = 4, 8
    for prefix in (2, 4, 6, 12, 40):
        s = sfi.init_decode_state(prefix, 1, 1, lim).per_layer[0]
        want = max(0, min(8, prefix - min(4, prefix)))
        assert s.recent_len == want
        if want:
            assert s.recent_start + s.recent_len - 1 == prefix


def test_flop_model():  # test_smoke.py:144-146
    assert sfi.flop_model(16384, 262, 0.0) == pytest.approx(62.5, abs=0.1)
    assert sfi.flop_model(4096, 4096, 0.5) == pytest.approx(1.0)

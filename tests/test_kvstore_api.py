"""The reference's attention-side KATs (test_attention.cpp) through the C++ host
API's KvStore / attention_kernel_dense / attention_kernel_sparse (pybind), all
of which run the sm_100a kernels."""
from __future__ import annotations

import numpy as np
import pytest

from helpers import bf16_round, oracle, rel_err, store_from_rows

pytestmark = pytest.mark.gpu


def _store(n_tokens, H=2, Hq=4, d=64, seed=3, ns=4, R=32, K=64, Lmax=512):
    import paper_2603_12038_b200 as sfi

    spec = sfi.ModelSpec()
    spec.n_layers, spec.n_query_heads, spec.n_kv_heads, spec.head_dim, spec.max_positions = 1, Hq, H, d, Lmax
    lim = sfi.CacheLimits()
    lim.n_sink, lim.n_recent, lim.k_budget = ns, R, K
    st = sfi.KvStore(spec, lim)
    rng = np.random.default_rng(seed)
    ks = bf16_round(rng.standard_normal((n_tokens, H * d)).astype(np.float32))
    vs = bf16_round(rng.standard_normal((n_tokens, H * d)).astype(np.float32))
    for t in range(n_tokens):
        st.begin_token()
        st.append_layer(0, ks[t].tolist(), vs[t].tolist())
        st.end_token()
    return sfi, st, ks, vs


def test_single_token_context_returns_v_exactly():  # test_attention.cpp:137-155
    sfi, st, ks, vs = _store(1)
    q = np.random.default_rng(1).standard_normal(4 * 64)
    out = np.asarray(sfi.attention_kernel_dense(st, 0, q.tolist()))
    G, d = 2, 64
    for qh in range(4):
        h = qh // G
        assert np.array_equal(out[qh * d:(qh + 1) * d], vs[0, h * d:(h + 1) * d].astype(np.float64))


def _support(sfi, L, ns, R, sel):
    sup = sfi.SupportSet()
    sup.sink = list(range(1, ns + 1))
    sup.selected = [list(map(int, s)) for s in sel]
    rl = min(R, L - ns)
    sup.recent_start, sup.recent_len = L - rl + 1, rl
    return sup


def test_full_support_sparse_equals_dense():  # test_attention.cpp:230-255
    sfi, st, ks, vs = _store(300, K=512)
    L, ns, R = 300, 4, 32
    J = list(range(ns + 1, L - min(R, L - ns) + 1))
    st.reorganize(0, list(range(1, ns + 1)), [J, J])
    q = np.random.default_rng(2).standard_normal(4 * 64).tolist()
    dense = np.asarray(sfi.attention_kernel_dense(st, 0, q))
    sparse = np.asarray(sfi.attention_kernel_sparse(st, 0, q, _support(sfi, L, ns, R, [J, J])))
    assert rel_err(sparse, dense) < 1e-5  # same support, fp32 summation order only


def test_sparse_matches_masked_oracle_and_reads_constant_in_L():  # :257-291, :350-387
    reads = []
    for L in (200, 400):
        sfi, st, ks, vs = _store(L, seed=L)
        ns, R = 4, 32
        rng = np.random.default_rng(L)
        J = np.arange(ns + 1, L - min(R, L - ns) + 1)
        sel = [np.sort(rng.choice(J, 60, replace=False)), np.sort(rng.choice(J, 60, replace=False))]
        st.reorganize(0, list(range(1, ns + 1)), [s.tolist() for s in sel])
        q = rng.standard_normal(4 * 64)
        stats = sfi.KernelStats()
        got = np.asarray(sfi.attention_kernel_sparse(st, 0, q.tolist(), _support(sfi, L, ns, R, sel), stats))
        k = np.transpose(ks.reshape(L, 2, 64), (1, 0, 2))
        v = np.transpose(vs.reshape(L, 2, 64), (1, 0, 2))
        orc_st = store_from_rows(oracle(), k, v, 4)
        orc_st.reorganize(0, list(range(1, ns + 1)), sel)
        want, _ = orc_st.attention_sparse(0, q, list(range(1, ns + 1)), sel, L - R + 1, R)
        assert rel_err(got, want) < 2e-3
        reads.append(stats.reads)
    assert reads[0] == reads[1] == 2 * (4 + 60 + 32)  # H * (sink + selected + recent), independent of L


def test_stale_compact_is_a_structured_error():  # test_attention.cpp:327-348
    sfi, st, ks, vs = _store(120)
    st.reorganize(0, [1, 2, 3, 4], [[10, 20], [11, 21]])
    q = np.zeros(4 * 64).tolist()
    with pytest.raises(sfi.SfiError) as e:
        sfi.attention_kernel_sparse(st, 0, q, _support(sfi, 120, 4, 32, [[10, 30], [11, 21]]))
    assert e.value.code == "stale_compact"

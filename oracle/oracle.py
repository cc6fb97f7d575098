"""CPU oracle loader — TEST INFRASTRUCTURE ONLY.

Loads oracle/_ref/libsfi_ref.so (the unmodified reference, built by
oracle/Makefile from /root/reference) or oracle/liboracle.so (the C
restatement, oracle/sfi_oracle.c); both implement oracle/oracle_abi.h.
Only tests/, __graft_entry__.smoke() and bench.py's CPU arms import this
module, and only as the checker / CPU baseline — never the product path.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libsfi_ref.so")
PORT_SO = os.path.join(HERE, "liboracle.so")

ERROR_NAMES = {
    1: "config", 2: "empty_support", 3: "support_mismatch", 4: "non_finite_input",
    5: "overlap_violation", 6: "stale_compact", 7: "out_of_range",
    8: "bad_weight_file", 9: "context_overflow", 10: "io",
}


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{ERROR_NAMES.get(code, code)}] {msg}")
        self.code = code
        self.name = ERROR_NAMES.get(code, str(code))


class SelectorCfg(C.Structure):
    _fields_ = [(n, C.c_double) for n in (
        "alpha", "gamma", "beta", "p_curve", "eta", "lambda_clip", "alpha_soft",
        "alpha_cross", "temperature", "epsilon")] + [
        ("nms_radius", C.c_int32), ("k_budget", C.c_int32), ("pool", C.c_int32)]


# selector defaults, config.hpp:31-47
DEFAULTS = dict(alpha=1.0, gamma=1.0, beta=1.0, p_curve=2.0, eta=0.5, lambda_clip=0.02,
                alpha_soft=0.5, alpha_cross=0.35, temperature=1.0, epsilon=1e-8,
                nms_radius=2, k_budget=2048, pool=0)


def make_cfg(**kw) -> SelectorCfg:
    d = dict(DEFAULTS)
    d.update(kw)
    return SelectorCfg(**d)


def build(ref: bool = True) -> None:
    """Builds the port (always) and the reference (when /root/reference exists)."""
    targets = ["port"]
    if ref and os.path.isdir("/root/reference/proj/src"):
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", HERE, *targets], check=True)


_P = np.ctypeslib.ndpointer


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


class ToySpec(C.Structure):
    _fields_ = [(n, C.c_int32) for n in ("n_layers", "n_query_heads", "n_kv_heads", "head_dim",
                                         "vocab_size", "max_positions")] + [("rope_base", C.c_double)]


class ToyLimits(C.Structure):
    _fields_ = [("n_sink", C.c_int32), ("n_recent", C.c_int32), ("k_budget", C.c_int32),
                ("trigger_tokens", C.c_void_p), ("n_trigger", C.c_int32), ("t_max", C.c_int32),
                ("window_prefill", C.c_int32)]


class Oracle:
    """One oracle library (kind 'reference' or 'port')."""

    def __init__(self, path: str):
        self.path = path
        self.lib = C.CDLL(path, mode=os.RTLD_LOCAL if hasattr(os, "RTLD_LOCAL") else 0)
        L = self.lib
        L.orc_kind.restype = C.c_char_p
        self.kind = L.orc_kind().decode()
        vp = C.c_void_p
        L.orc_store_create.restype = vp
        L.orc_store_create.argtypes = [C.c_int] * 5 + [C.c_char_p, C.c_int]
        L.orc_store_destroy.argtypes = [vp]
        L.orc_store_size.argtypes = [vp]
        L.orc_store_size.restype = C.c_int32
        L.orc_store_key_norm.argtypes = [vp, C.c_int, C.c_int, C.c_int32]
        L.orc_store_key_norm.restype = C.c_double
        L.orc_recent_window.argtypes = [C.c_int32, C.c_int, C.c_int, vp, vp]
        L.orc_recent_window.restype = None
        for name in ("orc_run_selector", "orc_select_top_k", "orc_refine_soft_nms",
                     "orc_refine_cross_head", "orc_store_append", "orc_store_append_many",
                     "orc_store_reorganize", "orc_store_compact", "orc_attention_dense",
                     "orc_attention_sparse", "orc_dense_capture"):
            getattr(L, name).restype = C.c_int
        if self.kind == "reference":  # toy model + request loop: reference library only
            L.orc_toy_checksum.restype = C.c_double
            L.orc_toy_checksum.argtypes = [C.c_void_p, C.c_uint64]
            L.orc_toy_run_request.restype = C.c_int
            L.orc_toy_run_dense.restype = C.c_int
            L.orc_toy_capture.restype = C.c_int

    # ---- toy model + request loop (reference only, scheduler.cpp:213-365) ----
    @staticmethod
    def _toy_spec(spec: dict) -> ToySpec:
        return ToySpec(**{k: spec[k] for k in ("n_layers", "n_query_heads", "n_kv_heads", "head_dim",
                                               "vocab_size", "max_positions")},
                       rope_base=float(spec.get("rope_base", 10000.0)))

    def toy_checksum(self, spec: dict, seed: int) -> float:
        ts = self._toy_spec(spec)
        return self.lib.orc_toy_checksum(C.byref(ts), C.c_uint64(seed))

    def toy_run_request(self, spec: dict, seed: int, prompt, limits: dict, cfg: SelectorCfg, max_new: int,
                        logits: bool = True):
        """Reference run_request; returns dict(tokens, slow, cause, logits [max_new][vocab])."""
        ts = self._toy_spec(spec)
        prompt = _i32(prompt)
        trig = _i32(limits.get("trigger_tokens", [0, 1, 2, 3, 4]))
        tl = ToyLimits(n_sink=limits.get("n_sink", 4), n_recent=limits.get("n_recent", 256),
                       k_budget=limits.get("k_budget", 2048), trigger_tokens=trig.ctypes.data,
                       n_trigger=len(trig), t_max=limits.get("t_max", 64),
                       window_prefill=limits.get("window_prefill", 16))
        tok = np.zeros(max_new, np.int32)
        slow = np.zeros(max_new, np.int32)
        cause = np.zeros(max_new, np.int32)
        lg = np.zeros((max_new, spec["vocab_size"]), np.float64) if logits else None
        L, H, K = spec["n_layers"], spec["n_kv_heads"], tl.k_budget
        sel = np.zeros((max_new, L, H, max(K, 1)), np.int32)
        nsel = np.zeros((max_new, L, H), np.int32)
        err = C.create_string_buffer(512)
        rc = self.lib.orc_toy_run_request(C.byref(ts), C.c_uint64(seed), _ptr(prompt), C.c_int(len(prompt)),
                                          C.byref(tl), C.byref(cfg), C.c_int(max_new), _ptr(tok), _ptr(slow),
                                          _ptr(cause), _ptr(lg), _ptr(sel), _ptr(nsel), err, C.c_int(512))
        self._check(rc, err)
        selected = [[[sel[i, l, h, : nsel[i, l, h]].tolist() for h in range(H)] for l in range(L)]
                    for i in range(max_new)]
        return dict(tokens=tok, slow=slow, cause=cause, logits=lg, selected=selected)

    def toy_run_dense(self, spec: dict, seed: int, prompt, max_new: int, logits: bool = True):
        ts = self._toy_spec(spec)
        prompt = _i32(prompt)
        tok = np.zeros(max_new, np.int32)
        lg = np.zeros((max_new, spec["vocab_size"]), np.float64) if logits else None
        err = C.create_string_buffer(512)
        rc = self.lib.orc_toy_run_dense(C.byref(ts), C.c_uint64(seed), _ptr(prompt), C.c_int(len(prompt)),
                                        C.c_int(max_new), _ptr(tok), _ptr(lg), err, C.c_int(512))
        self._check(rc, err)
        return dict(tokens=tok, logits=lg)

    def toy_capture(self, spec: dict, seed: int, tokens, allowed, pool: int = 0):
        """The reference run_step's own slow-step capture at the last token
        (layer 0): dict(logits [H][nJ], context [Hq*d], q [Hq*d] post-rotary,
        k, v [n][H*d] fp32 paged rows)."""
        ts = self._toy_spec(spec)
        tokens = _i32(tokens)
        allowed = _i32(allowed)
        n, nJ = len(tokens), len(allowed)
        H, Hq, d = spec["n_kv_heads"], spec["n_query_heads"], spec["head_dim"]
        lg = np.zeros((H, max(nJ, 1)), np.float64)
        ctx = np.zeros(Hq * d, np.float64)
        q = np.zeros(Hq * d, np.float64)
        k = np.zeros((n, H * d), np.float32)
        v = np.zeros((n, H * d), np.float32)
        err = C.create_string_buffer(512)
        rc = self.lib.orc_toy_capture(C.byref(ts), C.c_uint64(seed), _ptr(tokens), C.c_int(n), C.c_int(nJ),
                                      _ptr(allowed if nJ else _i32([0])), C.c_int(pool), _ptr(lg), _ptr(ctx),
                                      _ptr(q), _ptr(k), _ptr(v), err, C.c_int(512))
        self._check(rc, err)
        return dict(logits=lg[:, :nJ].copy(), context=ctx, q=q, k=k, v=v)

    def _check(self, rc: int, err) -> None:
        if rc:
            raise OracleError(rc, err.value.decode(errors="replace"))

    # ---- Selector -------------------------------------------------------
    def run_selector(self, values, allowed, norms, cfg: SelectorCfg | None = None,
                     width: int = 1, stages: bool = False):
        """values: [H][W*n] (or [H][n] for W=1); allowed: [n]; norms: [H][n].
        Returns (list of per-head ascending position arrays, stages dict)."""
        cfg = cfg or make_cfg()
        values = _f64(values)
        allowed = _i32(allowed)
        norms = _f64(norms)
        H = values.shape[0]
        n = allowed.shape[0]
        cap = max(1, min(cfg.k_budget, n))
        out = np.zeros((H, cap), np.int32)
        cnt = np.zeros(H, np.int32)
        st = {}
        if stages:
            for k in ("z_base", "z_nms", "z_adj", "evidence", "prior"):
                st[k] = np.zeros((H, n), np.float64)
            st["lambda"] = np.zeros(H, np.float64)
        err = C.create_string_buffer(512)
        rc = self.lib.orc_run_selector(
            C.c_int(H), C.c_int(width), C.c_int(n), _ptr(allowed), _ptr(values), _ptr(norms),
            C.byref(cfg), _ptr(out), C.c_int(cap), _ptr(cnt),
            _ptr(st.get("z_base")), _ptr(st.get("z_nms")), _ptr(st.get("z_adj")),
            _ptr(st.get("lambda")), _ptr(st.get("evidence")), _ptr(st.get("prior")),
            err, C.c_int(512))
        self._check(rc, err)
        return [out[h, : cnt[h]].copy() for h in range(H)], st

    def select_top_k(self, scores, allowed, k: int):
        scores = _f64(scores)
        allowed = _i32(allowed)
        n = scores.shape[0]
        out = np.zeros(max(1, min(max(k, 0), n)), np.int32)
        cnt = C.c_int32(0)
        err = C.create_string_buffer(512)
        rc = self.lib.orc_select_top_k(C.c_int(n), _ptr(scores), _ptr(allowed), C.c_int(k),
                                       _ptr(out), C.byref(cnt), err, C.c_int(512))
        self._check(rc, err)
        return out[: cnt.value].copy()

    def refine_soft_nms(self, z, cfg: SelectorCfg | None = None):
        cfg = cfg or make_cfg()
        z = _f64(z)
        out = np.zeros_like(z)
        err = C.create_string_buffer(512)
        self._check(self.lib.orc_refine_soft_nms(C.c_int(z.shape[0]), _ptr(z), C.byref(cfg),
                                                 _ptr(out), err, C.c_int(512)), err)
        return out

    def refine_cross_head(self, z, cfg: SelectorCfg | None = None):
        cfg = cfg or make_cfg()
        z = _f64(z)
        out = np.zeros_like(z)
        err = C.create_string_buffer(512)
        self._check(self.lib.orc_refine_cross_head(C.c_int(z.shape[0]), C.c_int(z.shape[1]),
                                                   _ptr(z), C.byref(cfg), _ptr(out), err,
                                                   C.c_int(512)), err)
        return out

    def recent_window(self, prefix_len: int, n_sink: int, n_recent: int):
        a, b = C.c_int32(0), C.c_int32(0)
        self.lib.orc_recent_window(C.c_int32(prefix_len), C.c_int(n_sink), C.c_int(n_recent),
                                   C.byref(a), C.byref(b))
        return a.value, b.value

    # ---- KV store -------------------------------------------------------
    def store(self, n_layers: int, n_kv_heads: int, n_q_heads: int, head_dim: int,
              max_positions: int) -> "Store":
        return Store(self, n_layers, n_kv_heads, n_q_heads, head_dim, max_positions)


class Store:
    """KvStore (attention.hpp:100-155) held by an oracle library."""

    def __init__(self, orc: Oracle, n_layers, H, Hq, d, max_positions):
        self.orc, self.n_layers, self.H, self.Hq, self.d = orc, n_layers, H, Hq, d
        err = C.create_string_buffer(512)
        self.h = orc.lib.orc_store_create(n_layers, H, Hq, d, max_positions, err, 512)
        if not self.h:
            raise OracleError(1, err.value.decode())

    def __del__(self):
        h = getattr(self, "h", None)
        if h:
            self.orc.lib.orc_store_destroy(C.c_void_p(h))
            self.h = None

    @property
    def size(self) -> int:
        return self.orc.lib.orc_store_size(C.c_void_p(self.h))

    def append(self, k, v):
        """k, v: [n_layers][H*d] fp32 for one token."""
        k, v = _f32(k), _f32(v)
        err = C.create_string_buffer(512)
        self.orc._check(self.orc.lib.orc_store_append(C.c_void_p(self.h), _ptr(k), _ptr(v), err, 512), err)

    def append_many(self, k, v):
        """One-layer stores: k, v: [count][H*d] fp32."""
        k, v = _f32(k), _f32(v)
        err = C.create_string_buffer(512)
        self.orc._check(self.orc.lib.orc_store_append_many(C.c_void_p(self.h), C.c_int(k.shape[0]),
                                                           _ptr(k), _ptr(v), err, 512), err)

    def key_norm(self, layer, head, pos) -> float:
        return self.orc.lib.orc_store_key_norm(C.c_void_p(self.h), layer, head, pos)

    @staticmethod
    def _flat(selected):
        counts = _i32([len(s) for s in selected])
        flat = _i32(np.concatenate([np.asarray(s, np.int32) for s in selected]) if
                    sum(len(s) for s in selected) else np.zeros(1, np.int32))
        return counts, flat

    def reorganize(self, layer, sink, selected):
        n_sink = len(sink)
        sink_a = _i32(sink if n_sink else np.zeros(1, np.int32))
        counts, flat = self._flat(selected)
        err = C.create_string_buffer(512)
        self.orc._check(self.orc.lib.orc_store_reorganize(
            C.c_void_p(self.h), layer, C.c_int(n_sink), _ptr(sink_a), _ptr(counts), _ptr(flat),
            err, 512), err)

    def compact(self, layer, head, cap=1 << 20):
        pos = np.zeros(cap, np.int32)
        k = np.zeros(cap * self.d, np.float32)
        v = np.zeros(cap * self.d, np.float32)
        cnt = C.c_int32(0)
        err = C.create_string_buffer(512)
        self.orc._check(self.orc.lib.orc_store_compact(C.c_void_p(self.h), layer, head, cap,
                                                       _ptr(pos), _ptr(k), _ptr(v), C.byref(cnt),
                                                       err, 512), err)
        n = cnt.value
        return pos[:n].copy(), k[: n * self.d].reshape(n, self.d).copy(), v[: n * self.d].reshape(n, self.d).copy()

    def attention_dense(self, layer, q):
        q = _f64(q).reshape(-1)
        out = np.zeros(self.Hq * self.d, np.float64)
        reads = C.c_uint64(0)
        err = C.create_string_buffer(512)
        self.orc._check(self.orc.lib.orc_attention_dense(C.c_void_p(self.h), layer, _ptr(q), _ptr(out),
                                                         C.byref(reads), err, 512), err)
        return out, reads.value

    def attention_sparse(self, layer, q, sink, selected, recent_start, recent_len):
        q = _f64(q).reshape(-1)
        n_sink = len(sink)
        sink_a = _i32(sink if n_sink else np.zeros(1, np.int32))
        counts, flat = self._flat(selected)
        out = np.zeros(self.Hq * self.d, np.float64)
        reads = C.c_uint64(0)
        err = C.create_string_buffer(512)
        self.orc._check(self.orc.lib.orc_attention_sparse(
            C.c_void_p(self.h), layer, _ptr(q), C.c_int(n_sink), _ptr(sink_a), _ptr(counts), _ptr(flat),
            C.c_int32(recent_start), C.c_int32(recent_len), _ptr(out), C.byref(reads), err, 512), err)
        return out, reads.value

    def dense_capture(self, layer, q, allowed, pool=0):
        q = _f64(q).reshape(-1)
        allowed = _i32(allowed)
        nJ = allowed.shape[0]
        out = np.zeros(self.Hq * self.d, np.float64)
        logits = np.zeros((self.H, max(nJ, 1)), np.float64)
        err = C.create_string_buffer(512)
        self.orc._check(self.orc.lib.orc_dense_capture(
            C.c_void_p(self.h), layer, _ptr(q), C.c_int(nJ), _ptr(allowed if nJ else _i32([0])),
            C.c_int(pool), _ptr(out), _ptr(logits), err, 512), err)
        return out, logits[:, :nJ].copy()



_CACHE: dict = {}


def load(kind: str = "best") -> Oracle:
    """kind: 'reference', 'port', or 'best' (reference when built, else port)."""
    if kind == "best":
        kind = "reference" if os.path.exists(REF_SO) else "port"
    if kind not in _CACHE:
        path = REF_SO if kind == "reference" else PORT_SO
        if not os.path.exists(path):
            if kind == "port":
                build(ref=False)
            else:
                raise FileNotFoundError(path)
        _CACHE[kind] = Oracle(path)
    return _CACHE[kind]


def have_reference() -> bool:
    return os.path.exists(REF_SO)

// bindings.cpp — pybind11 module `_sfi_b200`: the reference's `_sfi` names
// (proj/bindings/module.cpp:29-247, python/sfi/__init__.py) for the hot-path
// operators, backed by the B200 host API (namespace sfi), plus the batched
// device API (the C ABI one-to-one, taking raw device pointers and a
// cudaStream_t handle). The toy decoder / request loop bindings live in the
// test harness module (harness/toy_bindings.cpp -> _sfi_toy).
#include <pybind11/pybind11.h>
#include <pybind11/stl.h>

#include <cstdint>

#include "sfi_b200.h"
#include "sfi_b200.hpp"

namespace py = pybind11;
using namespace sfi;

namespace {

void* vp(std::uintptr_t p) { return reinterpret_cast<void*>(p); }

py::dict sizes_dict(const sfi_sizes& z) {
  py::dict d;
  d["kv_cache"] = z.kv_cache;
  d["key_norms"] = z.key_norms;
  d["compact"] = z.compact;
  d["sel"] = z.sel;
  d["n_sel"] = z.n_sel;
  d["per_batch"] = z.per_batch;
  d["workspace"] = z.workspace;
  d["pooled_logits"] = z.pooled_logits;
  return d;
}

}  // namespace

PYBIND11_MODULE(_sfi_b200, m) {
  m.doc() = "B200-native SFI decode-attention hot path (sm_100a)";

  static py::exception<Error> exc(m, "SfiError");
  py::register_exception_translator([](std::exception_ptr p) {
    try {
      if (p) std::rethrow_exception(p);
    } catch (const Error& e) {
      py::object type = py::reinterpret_borrow<py::object>(exc);
      py::object err = type(std::string("[") + error_code_name(e.code()) + "] " + e.what());
      err.attr("code") = error_code_name(e.code());
      PyErr_SetObject(exc.ptr(), err.ptr());
    }
  });

  py::enum_<PoolMode>(m, "PoolMode").value("mean", PoolMode::kMean).value("max", PoolMode::kMax);

  py::class_<SelectorConfig>(m, "SelectorConfig")
      .def(py::init<>())
      .def_readwrite("alpha", &SelectorConfig::alpha)
      .def_readwrite("gamma", &SelectorConfig::gamma)
      .def_readwrite("beta", &SelectorConfig::beta)
      .def_readwrite("p_curve", &SelectorConfig::p_curve)
      .def_readwrite("eta", &SelectorConfig::eta)
      .def_readwrite("lambda_clip", &SelectorConfig::lambda_clip)
      .def_readwrite("alpha_soft", &SelectorConfig::alpha_soft)
      .def_readwrite("alpha_cross", &SelectorConfig::alpha_cross)
      .def_readwrite("temperature", &SelectorConfig::temperature)
      .def_readwrite("nms_radius", &SelectorConfig::nms_radius)
      .def_readwrite("epsilon", &SelectorConfig::epsilon)
      .def_readwrite("k_budget", &SelectorConfig::k_budget)
      .def_readwrite("pool", &SelectorConfig::pool)
      .def("validate", &SelectorConfig::validate);

  py::class_<TriggerConfig>(m, "TriggerConfig")
      .def(py::init<>())
      .def_readwrite("trigger_tokens", &TriggerConfig::trigger_tokens)
      .def_readwrite("t_max", &TriggerConfig::t_max)
      .def_readwrite("window_decode", &TriggerConfig::window_decode)
      .def_readwrite("window_prefill", &TriggerConfig::window_prefill)
      .def("is_trigger", &TriggerConfig::is_trigger);

  py::class_<CacheLimits>(m, "CacheLimits")
      .def(py::init<>())
      .def_readwrite("n_sink", &CacheLimits::n_sink)
      .def_readwrite("n_recent", &CacheLimits::n_recent)
      .def_readwrite("k_budget", &CacheLimits::k_budget)
      .def("validate", &CacheLimits::validate);

  py::class_<Config>(m, "Config")
      .def(py::init<>())
      .def_readwrite("selector", &Config::selector)
      .def_readwrite("trigger", &Config::trigger)
      .def_readwrite("limits", &Config::limits)
      .def("validate", &Config::validate);
  m.def("default_config", &default_config);
  m.def("load_config_file", &load_config_file, py::arg("path"));
  m.def("save_config_file", &save_config_file, py::arg("config"), py::arg("path"));

  // distribution.hpp:31-58
  py::class_<ScoreDistribution>(m, "ScoreDistribution")
      .def(py::init<>())
      .def(py::init([](std::vector<Pos> support, std::vector<double> mass) {
             ScoreDistribution d;
             d.support = std::move(support);
             d.mass = std::move(mass);
             return d;
           }),
           py::arg("support"), py::arg("mass"))
      .def_readwrite("support", &ScoreDistribution::support)
      .def_readwrite("mass", &ScoreDistribution::mass);
  m.def("validate_distribution", &validate_distribution);
  m.def("normalize", [](const std::vector<Pos>& support, const std::vector<double>& weights) {
    return normalize(support, weights);
  });
  m.def("dot", &dot);
  m.def("squared_norm", &squared_norm);
  m.def("same_support", &same_support);

  py::class_<LogitWindow>(m, "LogitWindow")
      .def(py::init<>())
      .def_readwrite("width", &LogitWindow::width)
      .def_readwrite("allowed", &LogitWindow::allowed)
      .def_readwrite("values", &LogitWindow::values);

  py::class_<CacheStats>(m, "CacheStats")
      .def(py::init<>())
      .def_readwrite("key_norms", &CacheStats::key_norms)
      .def_readwrite("j_min", &CacheStats::j_min)
      .def_readwrite("j_max", &CacheStats::j_max)
      .def_readwrite("normalized_pos", &CacheStats::normalized_pos);
  m.def("make_cache_stats", &make_cache_stats, py::arg("key_norms"), py::arg("allowed"),
        py::arg("epsilon") = 1e-8);

  // selector.hpp:57-130: every stage on the device
  py::class_<FusedScore>(m, "FusedScore")
      .def_readonly("evidence", &FusedScore::evidence)
      .def_readonly("prior", &FusedScore::prior)
      .def_readonly("lambda_star", &FusedScore::lambda_star)
      .def_readonly("fused", &FusedScore::fused);
  py::class_<RefinedScores>(m, "RefinedScores")
      .def_readonly("base", &RefinedScores::base)
      .def_readonly("after_nms", &RefinedScores::after_nms)
      .def_readonly("after_cross", &RefinedScores::after_cross);
  py::class_<SelectorTrace>(m, "SelectorTrace")
      .def(py::init<>())
      .def_readwrite("capture_stages", &SelectorTrace::capture_stages)
      .def_readwrite("capture_debug", &SelectorTrace::capture_debug)
      .def_readonly("elementary_ops", &SelectorTrace::elementary_ops)
      .def_readonly("stages", &SelectorTrace::stages)
      .def_readonly("fusion", &SelectorTrace::fusion)
      .def_readonly("debug_lines", &SelectorTrace::debug_lines);
  m.def("evidence_from_window",
        [](const LogitWindow& w, const SelectorConfig& cfg) { return evidence_from_window(w, cfg); });
  m.def("prior_from_stats", [](const CacheStats& stats, const std::vector<Pos>& allowed,
                               const SelectorConfig& cfg) { return prior_from_stats(stats, allowed, cfg); });
  m.def("fuse", [](const ScoreDistribution& f, const ScoreDistribution& r, const SelectorConfig& cfg) {
    return fuse(f, r, cfg);
  });
  m.def("refine_soft_nms", [](const std::vector<double>& z, const SelectorConfig& cfg) { return refine_soft_nms(z, cfg); });
  m.def("refine_cross_head", [](const std::vector<std::vector<double>>& z, const SelectorConfig& cfg) {
    return refine_cross_head(z, cfg);
  });
  m.def("select_top_k", &select_top_k, py::arg("scores"), py::arg("allowed"), py::arg("k"));
  m.def(
      "run_selector",
      [](const LogitWindow& w, const CacheStats& stats, const SelectorConfig& cfg, SelectorTrace* trace) {
        return run_selector(w, stats, cfg, trace);
      },
      py::arg("window"), py::arg("stats"), py::arg("config"), py::arg("trace") = nullptr);

  py::class_<ModelSpec>(m, "ModelSpec")
      .def(py::init<>())
      .def_readwrite("n_layers", &ModelSpec::n_layers)
      .def_readwrite("n_query_heads", &ModelSpec::n_query_heads)
      .def_readwrite("n_kv_heads", &ModelSpec::n_kv_heads)
      .def_readwrite("head_dim", &ModelSpec::head_dim)
      .def_readwrite("vocab_size", &ModelSpec::vocab_size)
      .def_readwrite("max_positions", &ModelSpec::max_positions)
      .def_readwrite("rope_base", &ModelSpec::rope_base)
      .def("group_size", &ModelSpec::group_size)
      .def("validate", &ModelSpec::validate);

  py::class_<SupportSet>(m, "SupportSet")
      .def(py::init<>())
      .def_readwrite("sink", &SupportSet::sink)
      .def_readwrite("selected", &SupportSet::selected)
      .def_readwrite("recent_start", &SupportSet::recent_start)
      .def_readwrite("recent_len", &SupportSet::recent_len)
      .def("size_for_head", &SupportSet::size_for_head);

  py::class_<KernelStats>(m, "KernelStats")
      .def(py::init<>())
      .def_readwrite("flops", &KernelStats::flops)
      .def_readwrite("reads", &KernelStats::reads);

  py::class_<KvStore::CompactSegment>(m, "CompactSegment")
      .def_readonly("positions", &KvStore::CompactSegment::positions)
      .def_readonly("k", &KvStore::CompactSegment::k)
      .def_readonly("v", &KvStore::CompactSegment::v);

  py::class_<KvStore>(m, "KvStore")
      .def(py::init<const ModelSpec&, const CacheLimits&>(), py::arg("spec"),
           py::arg("limits") = CacheLimits{})
      .def("size", &KvStore::size)
      .def_property_readonly("spec", &KvStore::spec)
      .def("begin_token", &KvStore::begin_token)
      .def("append_layer",
           [](KvStore& s, int layer, const std::vector<float>& k, const std::vector<float>& v) {
             const size_t hd = static_cast<size_t>(s.spec().n_kv_heads) * s.spec().head_dim;
             if (k.size() != hd || v.size() != hd)
               fail(ErrorCode::kSupportMismatch, "append_layer: k/v must hold n_kv_heads * head_dim values");
             s.append_layer(layer, k.data(), v.data());
           })
      .def("end_token", &KvStore::end_token)
      .def("append_tokens",
           [](KvStore& s, int count, std::uintptr_t k, std::uintptr_t v) {
             s.append_tokens(count, reinterpret_cast<const float*>(k), reinterpret_cast<const float*>(v));
           },
           "host fp32 pointers [n_layers][count][H*d]")
      .def("key_row", &KvStore::key_row)
      .def("value_row", &KvStore::value_row)
      .def("key_at", &KvStore::key_row, "H*d values (copy of the view key_at returns)")
      .def("value_at", &KvStore::value_row)
      .def("set_access_trace", &KvStore::set_access_trace)
      .def("access_trace", [](KvStore& s) {
        py::list out;
        for (const auto& a : s.access_trace()) out.append(py::make_tuple(a.layer, a.head, a.slot));
        return out;
      })
      .def("key_norm", &KvStore::key_norm)
      .def("reorganize", &KvStore::reorganize)
      .def("compact_valid", &KvStore::compact_valid)
      .def("compact_matches", &KvStore::compact_matches)
      .def("compact", &KvStore::compact, py::return_value_policy::copy)
      .def("recent_tail", &KvStore::recent_tail);

  m.def("attention_kernel_dense",
        [](const KvStore& s, int layer, const std::vector<double>& q, KernelStats* stats) {
          return attention_kernel_dense(s, layer, q, stats);
        },
        py::arg("store"), py::arg("layer"), py::arg("q"), py::arg("stats") = nullptr);
  m.def("attention_kernel_sparse",
        [](const KvStore& s, int layer, const std::vector<double>& q, const SupportSet& sup,
           KernelStats* stats) { return attention_kernel_sparse(s, layer, q, sup, stats); },
        py::arg("store"), py::arg("layer"), py::arg("q"), py::arg("support"), py::arg("stats") = nullptr);
  py::class_<DenseCapture>(m, "DenseCapture")
      .def_readonly("context", &DenseCapture::context)
      .def_readonly("window", &DenseCapture::window);
  m.def("dense_capture", &dense_capture, py::arg("store"), py::arg("layer"), py::arg("q"),
        py::arg("allowed"), py::arg("pool") = PoolMode::kMean);

  py::class_<SparseState>(m, "SparseState")
      .def(py::init<>())
      .def_readwrite("layer", &SparseState::layer)
      .def_readwrite("sink", &SparseState::sink)
      .def_readwrite("recent_start", &SparseState::recent_start)
      .def_readwrite("recent_len", &SparseState::recent_len)
      .def_readwrite("selected", &SparseState::selected)
      .def("recent", &SparseState::recent)
      .def("support", &SparseState::support);
  py::class_<DecodeState>(m, "DecodeState")
      .def(py::init<>())
      .def_readwrite("t", &DecodeState::t)
      .def_readwrite("prefix_len", &DecodeState::prefix_len)
      .def_readwrite("g", &DecodeState::g)
      .def_readwrite("steps_since_slow", &DecodeState::steps_since_slow)
      .def_readwrite("last_token", &DecodeState::last_token)
      .def_readwrite("per_layer", &DecodeState::per_layer);
  m.def("init_decode_state", &init_decode_state, py::arg("prompt_len"), py::arg("n_layers"),
        py::arg("n_kv_heads"), py::arg("limits"));
  m.def("compute_allowed", &compute_allowed, py::arg("state"), py::arg("prefix_len"));
  m.def("next_step_type", &next_step_type, py::arg("state"), py::arg("trigger"));
  m.def("fast_step_update", &fast_step_update, py::arg("state"), py::arg("limits"));
  m.def("slow_step_update", &slow_step_update, py::arg("state"), py::arg("selected_per_layer"),
        py::arg("limits"));
  m.def("flop_model", &flop_model, py::arg("prefix_len"), py::arg("support"), py::arg("slow_fraction"));

  py::enum_<StepCause>(m, "StepCause")
      .value("initial", StepCause::kInitial)
      .value("trigger", StepCause::kTrigger)
      .value("forced", StepCause::kForced)
      .value("none", StepCause::kNone);
  py::class_<StepRecord>(m, "StepRecord")
      .def(py::init<>())
      .def_readwrite("t", &StepRecord::t)
      .def_readwrite("slow", &StepRecord::slow)
      .def_readwrite("cause", &StepRecord::cause)
      .def_readwrite("support_size", &StepRecord::support_size)
      .def_readwrite("allowed_size", &StepRecord::allowed_size)
      .def_readwrite("prefix_len", &StepRecord::prefix_len);
  m.def("step_record_to_json", &step_record_to_json);

  // ---- batched device API: the C ABI one-to-one --------------------------
  py::class_<sfi_shape>(m, "Shape")
      .def(py::init<>())
      .def_readwrite("n_layers", &sfi_shape::n_layers)
      .def_readwrite("batch", &sfi_shape::batch)
      .def_readwrite("n_kv_heads", &sfi_shape::n_kv_heads)
      .def_readwrite("n_q_heads", &sfi_shape::n_q_heads)
      .def_readwrite("head_dim", &sfi_shape::head_dim)
      .def_readwrite("max_positions", &sfi_shape::max_positions)
      .def_readwrite("n_sink", &sfi_shape::n_sink)
      .def_readwrite("k_budget", &sfi_shape::k_budget)
      .def_readwrite("n_recent", &sfi_shape::n_recent);

#define PTR_FIELD(name, type)                                                          \
  def_property(                                                                        \
      #name, [](const sfi_cache& c) { return reinterpret_cast<std::uintptr_t>(c.name); }, \
      [](sfi_cache& c, std::uintptr_t p) { c.name = reinterpret_cast<type>(p); })
  py::class_<sfi_cache>(m, "Cache")
      .def(py::init([]() { return sfi_cache{}; }))
      .PTR_FIELD(k_cache, void*)
      .PTR_FIELD(v_cache, void*)
      .PTR_FIELD(key_norms, double*)
      .PTR_FIELD(ck, void*)
      .PTR_FIELD(cv, void*)
      .PTR_FIELD(sel, int32_t*)
      .PTR_FIELD(n_sel, int32_t*)
      .PTR_FIELD(prefix_len, int32_t*)
      .PTR_FIELD(n_sink_b, int32_t*)
      .PTR_FIELD(recent_len, int32_t*)
      .PTR_FIELD(error_flags, uint32_t*)
      .PTR_FIELD(workspace, void*)
      .def_readwrite("workspace_bytes", &sfi_cache::workspace_bytes);
#undef PTR_FIELD

  py::class_<sfi_selector_params>(m, "SelectorParams")
      .def(py::init([](const SelectorConfig& c) { return to_params(c); }), py::arg("config") = SelectorConfig{});

  // ---- the C++ decode executor (sfi/decode.hpp): async slow step + graph-captured steps ----
  py::class_<DecodeExecutor>(m, "DecodeExecutor")
      .def(py::init([](const sfi_shape& s, const sfi_cache& c, std::uintptr_t stream, const SelectorConfig& cfg,
                       int slots, bool share_sm, std::uintptr_t logits_ring, int priorities) {
             return std::make_unique<DecodeExecutor>(s, c, vp(stream), cfg, slots, share_sm,
                                                     static_cast<float*>(vp(logits_ring)), priorities);
           }),
           py::arg("shape"), py::arg("cache"), py::arg("stream"), py::arg("selector") = SelectorConfig{},
           py::arg("slots") = 2, py::arg("share_sm") = true, py::arg("logits_ring") = 0,
           py::arg("priorities") = 0)
      .def("step",
           [](DecodeExecutor& x, bool slow, std::uintptr_t q, std::uintptr_t k, std::uintptr_t v, std::uintptr_t out,
              size_t sq, size_t skv, size_t so, bool rebuild_ring, std::vector<std::uintptr_t> wait_before,
              std::vector<std::uintptr_t> record_after, bool capture, std::uintptr_t origin,
              std::vector<std::uintptr_t> record_before_attention, std::vector<std::uintptr_t> aux_events) {
             StepBuffers io;
             io.q = static_cast<const float*>(vp(q));
             io.k_new = vp(k);
             io.v_new = vp(v);
             io.out = static_cast<float*>(vp(out));
             io.layer_stride_q = sq;
             io.layer_stride_kv = skv;
             io.layer_stride_out = so;
             StepHooks hooks;
             for (auto e : wait_before) hooks.wait_before.push_back(vp(e));
             for (auto e : record_after) hooks.record_after.push_back(vp(e));
             for (auto e : record_before_attention) hooks.record_before_attention.push_back(vp(e));
             // aux_events: [3][L] flattened (aux_begin, aux_selected, aux_end)
             if (!aux_events.empty()) {
               if (aux_events.size() % 3) throw std::invalid_argument("aux_events: 3 x n_layers events");
               const size_t L = aux_events.size() / 3;
               for (size_t i = 0; i < L; ++i) {
                 hooks.aux_begin.push_back(vp(aux_events[i]));
                 hooks.aux_selected.push_back(vp(aux_events[L + i]));
                 hooks.aux_end.push_back(vp(aux_events[2 * L + i]));
               }
             }
             const StepHooks* hp = (wait_before.empty() && record_after.empty() && record_before_attention.empty() &&
                                    aux_events.empty())
                                       ? nullptr
                                       : &hooks;
             if (capture) x.capture(slow, io, rebuild_ring, hp);
             else x.step(slow, io, rebuild_ring, hp, vp(origin));
           },
           py::arg("slow"), py::arg("q"), py::arg("k_new"), py::arg("v_new"), py::arg("out"), py::arg("stride_q") = 0,
           py::arg("stride_kv") = 0, py::arg("stride_out") = 0, py::arg("rebuild_ring") = false,
           py::arg("wait_before") = std::vector<std::uintptr_t>{}, py::arg("record_after") = std::vector<std::uintptr_t>{},
           py::arg("capture") = false, py::arg("origin") = 0,
           py::arg("record_before_attention") = std::vector<std::uintptr_t>{},
           py::arg("aux_events") = std::vector<std::uintptr_t>{})
      .def("replay", &DecodeExecutor::replay, py::arg("slow"))
      .def("captured", &DecodeExecutor::captured, py::arg("slow"))
      .def("logits_slot", [](const DecodeExecutor& x, int l) { return reinterpret_cast<std::uintptr_t>(x.logits_slot(l)); })
      .def("launches_per_step", &DecodeExecutor::launches_per_step, py::arg("slow"));

  m.def("launch_floor", [](int n, int grid, std::uintptr_t stream) { check(sfi_launch_floor(n, grid, vp(stream))); });
  m.def("version", &sfi_version);
  m.def("last_launch_count", &sfi_last_launch_count);
  m.def("buffer_sizes", [](const sfi_shape& s) {
    sfi_sizes z;
    check(sfi_buffer_sizes(&s, &z));
    return sizes_dict(z);
  });
  m.def("shape_validate", [](const sfi_shape& s) { check(sfi_shape_validate(&s)); });
  m.def("set_lengths", [](const sfi_shape& s, const sfi_cache& c, const std::vector<int32_t>& L,
                          const std::vector<int32_t>& nsb, py::object rl, std::uintptr_t stream) {
    if ((int)L.size() != s.batch || (int)nsb.size() != s.batch)
      fail(ErrorCode::kSupportMismatch, "set_lengths: one entry per request");
    if (rl.is_none()) {
      check(sfi_set_lengths(&s, &c, L.data(), nsb.data(), nullptr, vp(stream)));
    } else {
      auto r = rl.cast<std::vector<int32_t>>();
      if ((int)r.size() != s.batch) fail(ErrorCode::kSupportMismatch, "set_lengths: one entry per request");
      check(sfi_set_lengths(&s, &c, L.data(), nsb.data(), r.data(), vp(stream)));
    }
  });
  m.def("step_advance", [](const sfi_shape& s, const sfi_cache& c, std::uintptr_t stream) {
    check(sfi_step_advance(&s, &c, vp(stream)));
  });
  m.def("ring_append", [](const sfi_shape& s, const sfi_cache& c, int layer, std::uintptr_t k,
                          std::uintptr_t v, std::uintptr_t stream) {
    check(sfi_ring_append(&s, &c, layer, vp(k), vp(v), vp(stream)));
  });
  m.def("append_block", [](const sfi_shape& s, const sfi_cache& c, int layer, int count, std::uintptr_t k,
                           std::uintptr_t v, std::uintptr_t stream) {
    check(sfi_append_block(&s, &c, layer, count, vp(k), vp(v), vp(stream)));
  });
  m.def("dense_decode", [](const sfi_shape& s, const sfi_cache& c, int layer, std::uintptr_t q,
                           std::uintptr_t out, std::uintptr_t logits, int pool, std::uintptr_t stream) {
    check(sfi_dense_decode(&s, &c, layer, static_cast<const float*>(vp(q)), static_cast<float*>(vp(out)),
                           static_cast<float*>(vp(logits)), pool, vp(stream)));
  });
  m.def("sparse_decode", [](const sfi_shape& s, const sfi_cache& c, int layer, std::uintptr_t q,
                            std::uintptr_t out, std::uintptr_t stream) {
    check(sfi_sparse_decode(&s, &c, layer, static_cast<const float*>(vp(q)), static_cast<float*>(vp(out)),
                            vp(stream)));
  });
  m.def("dense_decode_ex", [](const sfi_shape& s, const sfi_cache& c, int layer, std::uintptr_t q,
                              std::uintptr_t out, std::uintptr_t lse, std::uintptr_t logits, int pool, int flags,
                              std::uintptr_t stream) {
    check(sfi_dense_decode_ex(&s, &c, layer, static_cast<const float*>(vp(q)), static_cast<float*>(vp(out)),
                              static_cast<float*>(vp(lse)), static_cast<float*>(vp(logits)), pool, flags, vp(stream)));
  });
  m.attr("DENSE_SHARE_SM") = SFI_DENSE_SHARE_SM;
  m.attr("DENSE_TC") = SFI_DENSE_TC;
  m.attr("DENSE_MMA") = SFI_DENSE_MMA;
  m.def("fast_decode", [](const sfi_shape& s, const sfi_cache& c, int layer, std::uintptr_t q,
                          std::uintptr_t k, std::uintptr_t v, std::uintptr_t out, int flags,
                          std::uintptr_t stream) {
    check(sfi_fast_decode(&s, &c, layer, static_cast<const float*>(vp(q)), vp(k), vp(v),
                          static_cast<float*>(vp(out)), flags, vp(stream)));
  });
  m.attr("FAST_PREFETCH") = SFI_FAST_PREFETCH;
  // sequence sharding (C4)
  m.def("seq_lengths", [](const sfi_shape& s, const sfi_cache& c, std::uintptr_t gp, std::uintptr_t gs,
                          std::uintptr_t gr, int advance, int base, int is_last, std::uintptr_t j_off,
                          std::uintptr_t n_glob, std::uintptr_t stream) {
    check(sfi_seq_lengths(&s, &c, static_cast<int32_t*>(vp(gp)), static_cast<const int32_t*>(vp(gs)),
                          static_cast<int32_t*>(vp(gr)), advance, base, is_last, static_cast<int32_t*>(vp(j_off)),
                          static_cast<int32_t*>(vp(n_glob)), vp(stream)));
  });
  m.def("dense_decode_partial", [](const sfi_shape& s, const sfi_cache& c, int layer, std::uintptr_t q,
                                   std::uintptr_t out, std::uintptr_t lse, std::uintptr_t logits, int pool,
                                   std::uintptr_t stream) {
    check(sfi_dense_decode_partial(&s, &c, layer, static_cast<const float*>(vp(q)), static_cast<float*>(vp(out)),
                                   static_cast<float*>(vp(lse)), static_cast<float*>(vp(logits)), pool, vp(stream)));
  });
  m.def("fast_decode_partial", [](const sfi_shape& s, const sfi_cache& c, int layer, std::uintptr_t q,
                                  std::uintptr_t k, std::uintptr_t v, std::uintptr_t out, std::uintptr_t lse,
                                  int flags, std::uintptr_t stream) {
    check(sfi_fast_decode_partial(&s, &c, layer, static_cast<const float*>(vp(q)), vp(k), vp(v),
                                  static_cast<float*>(vp(out)), static_cast<float*>(vp(lse)), flags, vp(stream)));
  });
  m.def("merge_partials", [](int n_parts, int rows, int d, std::uintptr_t o, std::uintptr_t lse, std::uintptr_t out,
                             std::uintptr_t stream) {
    check(sfi_merge_partials(n_parts, rows, d, static_cast<const float*>(vp(o)), static_cast<const float*>(vp(lse)),
                             static_cast<float*>(vp(out)), vp(stream)));
  });
  m.def("peer_publish", [](std::uintptr_t flag, std::uintptr_t stream) {
    check(sfi_peer_publish(static_cast<int32_t*>(vp(flag)), vp(stream)));
  });
  m.def("peer_gather", [](int n_parts, int64_t bytes, std::uintptr_t src_ptrs, std::uintptr_t flag_ptrs,
                          std::uintptr_t my_flag, std::uintptr_t dst, std::uintptr_t stream) {
    check(sfi_peer_gather(n_parts, bytes, static_cast<const void* const*>(vp(src_ptrs)),
                          static_cast<const int32_t* const*>(vp(flag_ptrs)), static_cast<const int32_t*>(vp(my_flag)),
                          vp(dst), vp(stream)));
  });
  m.def("peer_merge", [](int n_parts, int rows, int d, std::uintptr_t o_ptrs, std::uintptr_t lse_ptrs,
                         std::uintptr_t flag_ptrs, std::uintptr_t my_flag, std::uintptr_t out, std::uintptr_t stream) {
    check(sfi_peer_merge(n_parts, rows, d, static_cast<const float* const*>(vp(o_ptrs)),
                         static_cast<const float* const*>(vp(lse_ptrs)),
                         static_cast<const int32_t* const*>(vp(flag_ptrs)), static_cast<const int32_t*>(vp(my_flag)),
                         static_cast<float*>(vp(out)), vp(stream)));
  });
  m.def("seq_edges_doubles", [](const sfi_shape& s, const sfi_selector_params& prm) {
    return sfi_seq_edges_doubles(&s, &prm);
  });
  m.def("seq_pick_scratch_bytes", [](const sfi_shape& s, int n_shards) { return sfi_seq_pick_scratch_bytes(&s, n_shards); });
  m.def("seq_selector_stats", [](const sfi_shape& s, const sfi_cache& c, int layer, std::uintptr_t logits,
                                 const sfi_selector_params& prm, std::uintptr_t j_off, std::uintptr_t n_glob, int phase,
                                 std::uintptr_t row_stats, std::uintptr_t stats_all, int n_shards, std::uintptr_t edges,
                                 std::uintptr_t stream) {
    check(sfi_seq_selector_stats(&s, &c, layer, static_cast<const float*>(vp(logits)), &prm,
                                 static_cast<const int32_t*>(vp(j_off)), static_cast<const int32_t*>(vp(n_glob)), phase,
                                 static_cast<double*>(vp(row_stats)), static_cast<const double*>(vp(stats_all)),
                                 n_shards, static_cast<double*>(vp(edges)), vp(stream)));
  });
  m.def("seq_selector_finish", [](const sfi_shape& s, const sfi_cache& c, int layer, const sfi_selector_params& prm,
                                  std::uintptr_t j_off, std::uintptr_t n_glob, std::uintptr_t edges_all, int n_shards,
                                  int pos_base, std::uintptr_t cs, std::uintptr_t cp, std::uintptr_t stream) {
    check(sfi_seq_selector_finish(&s, &c, layer, &prm, static_cast<const int32_t*>(vp(j_off)),
                                  static_cast<const int32_t*>(vp(n_glob)), static_cast<const double*>(vp(edges_all)),
                                  n_shards, pos_base, static_cast<double*>(vp(cs)), static_cast<int32_t*>(vp(cp)),
                                  vp(stream)));
  });
  m.def("seq_selector_pick", [](const sfi_shape& s, const sfi_cache& c, int layer, int n_shards, std::uintptr_t cs,
                                std::uintptr_t cp, int pos_base, int pos_end, std::uintptr_t scratch,
                                std::uintptr_t stream) {
    check(sfi_seq_selector_pick(&s, &c, layer, n_shards, static_cast<const double*>(vp(cs)),
                                static_cast<const int32_t*>(vp(cp)), pos_base, pos_end, vp(scratch), vp(stream)));
  });
  m.def("prefill_capture", [](const sfi_shape& s, const sfi_cache& c, int layer, std::uintptr_t q, int W,
                              std::uintptr_t q_pos, std::uintptr_t out, int pool, std::uintptr_t stream) {
    check(sfi_prefill_capture(&s, &c, layer, static_cast<const float*>(vp(q)), W,
                              static_cast<const int32_t*>(vp(q_pos)), static_cast<float*>(vp(out)), pool, vp(stream)));
  });
  m.def("selector_window", [](const sfi_shape& s, const sfi_cache& c, int layer, std::uintptr_t logits, int W,
                              const sfi_selector_params& prm, std::uintptr_t stream) {
    check(sfi_selector_window(&s, &c, layer, static_cast<const float*>(vp(logits)), W, &prm, vp(stream)));
  });
  m.def("selector_fuse", [](const sfi_shape& s, const sfi_cache& c, int layer, std::uintptr_t logits,
                            const sfi_selector_params& prm, std::uintptr_t stream) {
    const double* z = nullptr;
    size_t bytes = 0;
    check(sfi_selector_fuse(&s, &c, layer, static_cast<const float*>(vp(logits)), &prm, &z, &bytes, vp(stream)));
    return py::make_tuple(reinterpret_cast<std::uintptr_t>(z), bytes);
  });
  m.def("selector_finish", [](const sfi_shape& s, const sfi_cache& c, int layer, const sfi_selector_params& prm,
                              std::uintptr_t z_all, int n_shards, int shard, std::uintptr_t stream) {
    check(sfi_selector_finish(&s, &c, layer, &prm, static_cast<const double*>(vp(z_all)), n_shards, shard,
                              vp(stream)));
  });
  // multi-GPU entry points over an NCCL communicator (ncclComm_t as an integer)
  m.def("selector_sharded_nccl", [](const sfi_shape& s, const sfi_cache& c, int layer, std::uintptr_t logits,
                                    const sfi_selector_params& prm, std::uintptr_t comm, int n_shards, int shard,
                                    std::uintptr_t z_all, std::uintptr_t stream) {
    check(sfi_selector_sharded_nccl(&s, &c, layer, static_cast<const float*>(vp(logits)), &prm, vp(comm), n_shards,
                                    shard, static_cast<double*>(vp(z_all)), vp(stream)));
  });
  m.def("merge_partials_nccl", [](int n_parts, int rows, int d, std::uintptr_t o, std::uintptr_t lse,
                                  std::uintptr_t o_all, std::uintptr_t lse_all, std::uintptr_t out,
                                  std::uintptr_t comm, std::uintptr_t stream) {
    check(sfi_merge_partials_nccl(n_parts, rows, d, static_cast<const float*>(vp(o)),
                                  static_cast<const float*>(vp(lse)), static_cast<float*>(vp(o_all)),
                                  static_cast<float*>(vp(lse_all)), static_cast<float*>(vp(out)), vp(comm),
                                  vp(stream)));
  });
  m.def("seq_selector_nccl_scratch_bytes", [](const sfi_shape& s, const sfi_selector_params& prm, int n_shards) {
    return sfi_seq_selector_nccl_scratch_bytes(&s, &prm, n_shards);
  });
  m.def("seq_selector_nccl", [](const sfi_shape& s, const sfi_cache& c, int layer, std::uintptr_t logits,
                                const sfi_selector_params& prm, std::uintptr_t j_off, std::uintptr_t n_glob,
                                int pos_base, int pos_end, std::uintptr_t comm, int n_shards, std::uintptr_t scratch,
                                size_t scratch_bytes, std::uintptr_t stream) {
    check(sfi_seq_selector_nccl(&s, &c, layer, static_cast<const float*>(vp(logits)), &prm,
                                static_cast<const int32_t*>(vp(j_off)), static_cast<const int32_t*>(vp(n_glob)),
                                pos_base, pos_end, vp(comm), n_shards, vp(scratch), scratch_bytes, vp(stream)));
  });
  m.def("selector", [](const sfi_shape& s, const sfi_cache& c, int layer, std::uintptr_t logits,
                       const sfi_selector_params& prm, std::uintptr_t stream) {
    check(sfi_selector(&s, &c, layer, static_cast<const float*>(vp(logits)), &prm, vp(stream)));
  });
  m.def("compact_build", [](const sfi_shape& s, const sfi_cache& c, int layer, int rebuild_ring,
                            std::uintptr_t stream) {
    check(sfi_compact_build(&s, &c, layer, rebuild_ring, vp(stream)));
  });
  m.def("read_errors", [](const sfi_cache& c, std::uintptr_t stream) {
    uint32_t flags = 0;
    const int rc = sfi_read_errors(&c, &flags, vp(stream));
    return py::make_tuple(rc, flags, std::string(rc ? sfi_last_error() : ""));
  });
  m.def("fill_synthetic", [](const sfi_shape& s, const sfi_cache& c, std::uint64_t seed, int len,
                             std::uintptr_t stream) {
    check(sfi_fill_synthetic(&s, &c, seed, len, vp(stream)));
  });
  m.def("selector_stages", [](const sfi_shape& s, const sfi_cache& c, int b, int n_j, std::uintptr_t stream) {
    std::vector<double> zb(static_cast<size_t>(s.n_kv_heads) * n_j), za(zb.size());
    check(sfi_selector_stages(&s, &c, b, zb.data(), za.data(), n_j, vp(stream)));
    return py::make_tuple(zb, za);
  });
}

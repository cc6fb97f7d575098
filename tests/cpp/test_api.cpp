// test_api.cpp — the reference's C++ call sites against include/sfi/*.hpp (the
// reference's header paths and namespace) and libsfi_b200.so.
// Restates KATs of /root/reference/proj/tests (test_core.cpp, test_scheduler.cpp,
// test_attention.cpp, test_selector.cpp) with a minimal self-contained checker.
// `test_api` runs the host-side cases; `test_api gpu` adds the device cases.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <random>
#include <sstream>
#include <string>
#include <vector>

// The reference's own header paths and namespace: a reference caller compiles
// unchanged against include/sfi/*.hpp and links libsfi_b200.so.
#include "sfi/attention.hpp"
#include "sfi/config.hpp"
#include "sfi/distribution.hpp"
#include "sfi/error.hpp"
#include "sfi/scheduler.hpp"
#include "sfi/selector.hpp"
#include "sfi_b200.h"

namespace {

int g_fail = 0, g_checks = 0;
#define CHECK(c)                                                           \
  do {                                                                     \
    ++g_checks;                                                            \
    if (!(c)) {                                                            \
      ++g_fail;                                                            \
      std::fprintf(stderr, "%s:%d: CHECK(%s) failed\n", __FILE__, __LINE__, #c); \
    }                                                                      \
  } while (0)
#define CHECK_THROWS_CODE(expr, code_)              \
  do {                                              \
    bool thrown_ = false;                           \
    try {                                           \
      expr;                                         \
    } catch (const sfi::Error& e_) {           \
      thrown_ = e_.code() == (code_);               \
    }                                               \
    CHECK(thrown_);                                 \
  } while (0)

using namespace sfi;

void test_default_config() {  // test_core.cpp:20-44
  const Config c = default_config();
  CHECK(c.selector.alpha == 1.0 && c.selector.gamma == 1.0 && c.selector.beta == 1.0);
  CHECK(c.selector.p_curve == 2.0 && c.selector.eta == 0.5 && c.selector.lambda_clip == 0.02);
  CHECK(c.selector.alpha_soft == 0.5 && c.selector.alpha_cross == 0.35 && c.selector.temperature == 1.0);
  CHECK(c.selector.nms_radius == 2 && c.selector.epsilon == 1e-8 && c.selector.k_budget == 2048);
  CHECK(c.limits.n_sink == 4 && c.limits.n_recent == 256 && c.limits.k_budget == 2048);
  CHECK(c.trigger.t_max == 64 && c.trigger.window_prefill == 16);
  SelectorConfig bad;
  bad.alpha = 0.0;
  CHECK_THROWS_CODE(bad.validate(), ErrorCode::kConfig);
}

void test_compute_allowed() {  // test_scheduler.cpp:68-83
  SparseState s;
  s.sink = {1};
  s.recent_start = 8;
  s.recent_len = 3;
  CHECK(compute_allowed(s, 10) == (std::vector<Pos>{2, 3, 4, 5, 6, 7}));
  SparseState all;
  all.sink = {1, 2};
  all.recent_start = 3;
  all.recent_len = 4;
  CHECK(compute_allowed(all, 6).empty());
  SparseState none;
  CHECK(compute_allowed(none, 4) == (std::vector<Pos>{1, 2, 3, 4}));
}

void test_triggers() {  // test_scheduler.cpp:85-124
  CacheLimits limits;
  limits.n_sink = 2;
  limits.n_recent = 4;
  TriggerConfig trig;
  trig.trigger_tokens = {9};
  DecodeState st = init_decode_state(16, 1, 1, limits);
  st.t = 1;
  st.last_token = 9;
  CHECK(next_step_type(st, trig) == 1);
  st.last_token = 5;
  st.steps_since_slow = 3;
  CHECK(next_step_type(st, trig) == 0);
  limits.n_sink = 1;
  DecodeState s2 = init_decode_state(8, 1, 1, limits);
  s2.last_token = 1;
  int forced = -1;
  for (int step = 1; step <= 70 && forced < 0; ++step) {
    if (next_step_type(s2, trig) == 1) {
      forced = step;
      CHECK(s2.steps_since_slow == 63);
      slow_step_update(s2, {{{}}}, limits);
      CHECK(s2.steps_since_slow == 0);
    } else {
      fast_step_update(s2, limits);
    }
  }
  CHECK(forced == 64);
}

void test_c_abi_errors() {
  sfi_shape s{};
  CHECK(sfi_shape_validate(&s) == SFI_ERR_CONFIG);
  s = sfi_shape{2, 1, 2, 6, 128, 64, 4, 8, 8};  // group 3: no kernel instantiation
  CHECK(sfi_shape_validate(&s) == SFI_ERR_UNSUPPORTED);
  s.n_q_heads = 5;  // not a multiple of the KV heads
  CHECK(sfi_shape_validate(&s) == SFI_ERR_CONFIG);
  s.n_q_heads = 32;  // group 16
  CHECK(sfi_shape_validate(&s) == SFI_OK);
  CHECK_THROWS_CODE(check(SFI_ERR_OVERLAP_VIOLATION), ErrorCode::kOverlapViolation);
}

// ------------------------------------------------------------------ GPU ----

ModelSpec spec64() {
  ModelSpec m;
  m.n_layers = 2;
  m.n_query_heads = 4;
  m.n_kv_heads = 2;
  m.head_dim = 64;
  m.max_positions = 256;
  return m;
}

std::vector<float> bf16_values(std::mt19937_64& rng, int n) {
  std::normal_distribution<float> nd(0.f, 1.f);
  std::vector<float> x(n);
  for (auto& v : x) {  // round to bf16 so the device copy is exact
    float f = nd(rng);
    uint32_t u;
    std::memcpy(&u, &f, 4);
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000u;
    std::memcpy(&v, &u, 4);
  }
  return x;
}

void test_reorganize_device() {  // test_attention.cpp:293-325
  const ModelSpec spec = spec64();
  CacheLimits limits;
  limits.n_sink = 4;
  limits.n_recent = 8;
  limits.k_budget = 16;
  KvStore store(spec, limits);
  std::mt19937_64 rng(2);
  const int n = 30, hd = spec.n_kv_heads * spec.head_dim;
  for (int t = 0; t < n; ++t) {
    store.begin_token();
    for (int l = 0; l < spec.n_layers; ++l) {
      const auto k = bf16_values(rng, hd), v = bf16_values(rng, hd);
      store.append_layer(l, k.data(), v.data());
    }
    store.end_token();
  }
  CHECK(store.size() == n);
  const std::vector<Pos> sink = {1, 2, 3};
  std::vector<std::vector<Pos>> selected = {{7, 11, 19}, {5, 11}};
  store.reorganize(0, sink, selected);
  const auto seg0 = store.compact(0, 0);
  CHECK(seg0.positions == (std::vector<Pos>{1, 2, 3, 7, 11, 19}));
  bool same = true;
  for (std::size_t i = 0; i < seg0.positions.size(); ++i) {
    const float* row = store.key_at(0, seg0.positions[i]);
    for (int c = 0; c < spec.head_dim; ++c) same &= seg0.k[i * spec.head_dim + c] == row[c];
  }
  CHECK(same);
  CHECK(store.compact(0, 1).positions == (std::vector<Pos>{1, 2, 3, 5, 11}));
  const auto k_before = seg0.k;
  store.reorganize(0, sink, selected);
  CHECK(store.compact(0, 0).k == k_before);
  store.reorganize(0, sink, {{}, {}});
  CHECK(store.compact(0, 0).positions == sink);
  CHECK_THROWS_CODE(store.reorganize(0, sink, {{500}, {}}), ErrorCode::kOutOfRange);
  bool overlap = false;
  try {
    store.reorganize(0, sink, {{3}, {}});
  } catch (const Error&) {
    overlap = true;
  }
  CHECK(overlap);
}

void test_selector_device() {  // test_selector.cpp:52-60, 295-301
  LogitWindow w;
  w.width = 1;
  w.allowed = {1, 2};
  w.values = {{0.0, std::log(2.0)}};
  const CacheStats st = make_cache_stats({{1.0, 1.0}}, w.allowed, 1e-8);
  SelectorConfig cfg;
  cfg.k_budget = 1;
  const auto sel = run_selector(w, st, cfg);
  CHECK(sel.size() == 1 && sel[0] == (std::vector<Pos>{2}));
  CHECK(select_top_k({0.1, 0.9, 0.5, 0.9}, {10, 20, 30, 40}, 2) == (std::vector<Pos>{20, 40}));
  CHECK(select_top_k({0.9, 0.5, 0.5}, {10, 20, 30}, 2) == (std::vector<Pos>{10, 20}));
  CHECK(select_top_k({0.9, 0.5}, {10, 20}, 0).empty());
  CHECK(select_top_k({0.1, 0.2}, {10, 20}, 5) == (std::vector<Pos>{10, 20}));
}


void test_kvstore_reference_surface() {  // attention.hpp:100-155 signatures and semantics
  const ModelSpec spec = spec64();
  KvStore store(spec);  // the reference constructor (default CacheLimits)
  std::mt19937_64 rng(5);
  const int n = 40, hd = spec.n_kv_heads * spec.head_dim;
  std::vector<std::vector<float>> keys;
  for (int t = 0; t < n; ++t) {
    store.begin_token();
    for (int l = 0; l < spec.n_layers; ++l) {
      const auto k = bf16_values(rng, hd), v = bf16_values(rng, hd);
      store.append_layer(l, k.data(), v.data());
      if (l == 1) keys.push_back(k);
    }
    store.end_token();
  }
  // key_at: a view of H*d floats in the reference's [pos][H][d] paged layout
  const float* k7 = store.key_at(1, 7);
  CHECK(std::equal(k7, k7 + hd, keys[6].begin()));
  CHECK_THROWS_CODE(store.key_at(0, n + 1), ErrorCode::kOutOfRange);
  double acc = 0.0;
  for (int c = 0; c < spec.head_dim; ++c) acc += static_cast<double>(keys[6][spec.head_dim + c]) * keys[6][spec.head_dim + c];
  CHECK(store.key_norm(1, 1, 7) == std::sqrt(acc));
  // a sink other than {1..n_sink}: gathered into the layer's own compact view
  const std::vector<Pos> sink = {2, 5};
  store.reorganize(1, sink, {{9, 30}, {3, 4, 6}});
  const KvStore::CompactSegment& seg = store.compact(1, 0);  // const reference, as in the reference
  CHECK(seg.positions == (std::vector<Pos>{2, 5, 9, 30}));
  bool same = true;
  for (std::size_t i = 0; i < seg.positions.size(); ++i) {
    const float* row = store.key_at(1, seg.positions[i]);
    for (int c = 0; c < spec.head_dim; ++c) same &= seg.k[i * spec.head_dim + c] == row[c];
  }
  CHECK(same);
  CHECK(store.compact_matches(1, sink, {{9, 30}, {3, 4, 6}}));
  // compact-read instrumentation (attention.cpp:242-244): one record per compact row per q head
  store.set_access_trace(true);
  SupportSet sup;
  sup.sink = sink;
  sup.selected = {{9, 30}, {3, 4, 6}};
  sup.recent_start = 31;  // a recent range that does not end at size()
  sup.recent_len = 4;
  std::vector<double> q(static_cast<std::size_t>(spec.n_query_heads) * spec.head_dim, 0.01);
  KernelStats ks;
  const auto out = attention_kernel_sparse(store, 1, q, sup, &ks);
  CHECK(out.size() == q.size() && ks.reads == static_cast<std::uint64_t>(4 + 4 + 5 + 4));
  const int G = spec.group_size();
  CHECK(store.access_trace().size() == static_cast<std::size_t>(G * (4 + 5)));
  CHECK(store.access_trace().front().layer == 1 && store.access_trace().back().head == 1);
}

void test_selector_stages_device() {  // selector.hpp:84-122 through the stage kernels
  LogitWindow w;
  w.width = 1;
  w.allowed = {5, 9};
  w.values = {{0.0, std::log(2.0)}};
  SelectorConfig cfg;
  const auto f = evidence_from_window(w, cfg);  // test_selector.cpp:52-60
  CHECK(f.size() == 1 && std::abs(f[0].mass[0] - 1.0 / 3) < 1e-12 && std::abs(f[0].mass[1] - 2.0 / 3) < 1e-12);
  CHECK(validate_distribution(f[0]));
  ScoreDistribution a, b;  // fuse KAT (test_selector.cpp:160-170)
  a.support = b.support = {1, 2, 3};
  a.mass = {0.5, 0.3, 0.2};
  b.mass = {1.0 / 3, 1.0 / 3, 1.0 / 3};
  const FusedScore fs = fuse(a, b, cfg);
  CHECK(fs.lambda_star == 0.02);
  CHECK(std::abs(fs.fused.mass[0] - 0.4966666666666667) < 1e-15);
  SelectorConfig r1;
  r1.nms_radius = 1;
  const auto nms = refine_soft_nms({1.0, 0.5, 0.2}, r1);  // test_selector.cpp:217-229
  CHECK(std::abs(nms[0] - 1.0) < 1e-15 && std::abs(nms[1] - 0.25) < 1e-15 && std::abs(nms[2] - 0.05) < 1e-15);
  const auto ch = refine_cross_head({{1.0}, {1.0}}, cfg);  // test_selector.cpp:261-280
  CHECK(std::abs(ch[0][0] - (1.0 + 0.35 * std::log(0.5))) < 1e-15);
  const std::vector<Pos> sup = {1, 2};
  const std::vector<double> wts = {1.0, 3.0};
  const ScoreDistribution nd = normalize(sup, wts);
  CHECK(nd.mass[0] == 0.25 && nd.mass[1] == 0.75);
  CHECK_THROWS_CODE(normalize(sup, std::vector<double>{0.0, 0.0}), ErrorCode::kEmptySupport);
  SelectorTrace trace;
  trace.capture_stages = true;
  const CacheStats st = make_cache_stats({{1.0, 1.0}}, w.allowed, 1e-8);
  const auto sel = run_selector(w, st, cfg, &trace);
  CHECK(sel[0].size() == 2 && trace.stages.base.size() == 1 && trace.fusion.size() == 1);
  CHECK(trace.elementary_ops > 0);
}

void test_config_io() {  // config.cpp:111-200
  Config c = default_config();
  c.selector.alpha_cross = 0.125;
  c.trigger.trigger_tokens = {7, 8};
  std::stringstream ss;
  save_config(c, ss);
  const Config back = load_config(ss);
  CHECK(back.selector.alpha_cross == 0.125 && back.trigger.trigger_tokens == (std::vector<TokenId>{7, 8}));
  std::stringstream bad("alpha=1\nbogus=2\n");
  CHECK_THROWS_CODE(load_config(bad), ErrorCode::kConfig);
}

}  // namespace

int main(int argc, char** argv) {
  const bool gpu = argc > 1 && std::string(argv[1]) == "gpu";
  std::vector<std::pair<const char*, std::function<void()>>> cases = {
      {"default_config", test_default_config},
      {"compute_allowed", test_compute_allowed},
      {"triggers", test_triggers},
      {"c_abi_errors", test_c_abi_errors},
      {"config_io", test_config_io},
  };
  if (gpu) {
    cases.push_back({"reorganize_device", test_reorganize_device});
    cases.push_back({"selector_device", test_selector_device});
    cases.push_back({"kvstore_reference_surface", test_kvstore_reference_surface});
    cases.push_back({"selector_stages_device", test_selector_stages_device});
  }
  for (auto& [name, fn] : cases) {
    const int before = g_fail;
    try {
      fn();
    } catch (const std::exception& e) {
      ++g_fail;
      std::fprintf(stderr, "%s: unexpected exception: %s\n", name, e.what());
    }
    std::printf("%s %s\n", g_fail == before ? "ok  " : "FAIL", name);
  }
  std::printf("%d checks, %d failed\n", g_checks, g_fail);
  return g_fail ? 1 : 0;
}

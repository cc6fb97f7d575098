// test_api.cpp — the reference's C++ call sites against include/sfi_b200.hpp.
// Restates KATs of /root/reference/proj/tests (test_core.cpp, test_scheduler.cpp,
// test_attention.cpp, test_selector.cpp) with a minimal self-contained checker.
// `test_api` runs the host-side cases; `test_api gpu` adds the device cases.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <random>
#include <string>
#include <vector>

#include "sfi_b200.hpp"

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
    } catch (const sfi_b200::Error& e_) {           \
      thrown_ = e_.code() == (code_);               \
    }                                               \
    CHECK(thrown_);                                 \
  } while (0)

using namespace sfi_b200;

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
    const auto row = store.key_row(0, seg0.positions[i]);
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

}  // namespace

// The reference's run_request / run_dense call sites (scheduler.hpp:116-135)
// against the device-path loop: C7 full retention (SFI tokens == dense tokens)
// and the C8 schedule rule, through the C++ API.
void test_request_loop_device() {
  ModelSpec spec;
  spec.n_layers = 2;
  spec.n_query_heads = 8;
  spec.n_kv_heads = 2;
  spec.head_dim = 64;
  spec.vocab_size = 256;
  spec.max_positions = 1024;
  const ToyModel model = ToyModel::random(spec, 9001);
  std::vector<TokenId> prompt;
  for (int i = 0; i < 70; ++i) prompt.push_back(5 + (i * 37) % 250);
  CacheLimits full;
  full.n_recent = 512;
  full.k_budget = 64;
  TriggerConfig trig;
  trig.t_max = 8;
  SelectorConfig cfg;
  cfg.k_budget = 64;
  const RequestResult r = run_request(model, prompt, full, trig, cfg, 24);
  const DenseResult d = run_dense(model, prompt, 24);
  CHECK(r.tokens.size() == 24 && r.log.size() == 24);
  CHECK(r.tokens == d.tokens);  // C7 (acceptance.cpp:125-160)
  int fast = 0, last_slow = 0;
  for (int t = 0; t < 24; ++t) {  // C8 rule (acceptance.cpp:162-205)
    const bool slow = t == 0 || trig.is_trigger(r.tokens[t - 1]) || t - last_slow >= trig.t_max;
    if (slow) last_slow = t;
    CHECK(slow == r.log[t].slow);
    fast += !r.log[t].slow;
  }
  CHECK(fast > 0);
  CHECK(r.total_kv_reads <= r.dense_equiv_reads);
  CacheLimits small;
  small.n_recent = 16;
  small.k_budget = 64;
  CHECK_THROWS_CODE(run_request(model, prompt, small, trig, SelectorConfig{}, 4), ErrorCode::kUnsupported);  // k mismatch
}

int main(int argc, char** argv) {
  const bool gpu = argc > 1 && std::string(argv[1]) == "gpu";
  std::vector<std::pair<const char*, std::function<void()>>> cases = {
      {"default_config", test_default_config},
      {"compute_allowed", test_compute_allowed},
      {"triggers", test_triggers},
      {"c_abi_errors", test_c_abi_errors},
  };
  if (gpu) {
    cases.push_back({"reorganize_device", test_reorganize_device});
    cases.push_back({"selector_device", test_selector_device});
    cases.push_back({"request_loop_device", test_request_loop_device});
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

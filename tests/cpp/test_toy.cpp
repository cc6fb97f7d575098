// test_toy.cpp — the reference's run_request / run_dense call sites against the
// TEST HARNESS (harness/sfi_toy.hpp, libsfi_toy.so) over libsfi_b200.so: the
// acceptance C7 / C8 checks through the C++ API, on the B200.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <random>
#include <string>
#include <vector>

#include "sfi_b200.hpp"
#include "sfi_toy.hpp"

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

int main() {
  try {
    test_request_loop_device();
  } catch (const std::exception& e) {
    ++g_fail;
    std::fprintf(stderr, "unexpected exception: %s\n", e.what());
  }
  std::printf("%d checks, %d failed\n", g_checks, g_fail);
  return g_fail ? 1 : 0;
}

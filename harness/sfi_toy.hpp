// harness/sfi_toy.hpp — END-TO-END TEST HARNESS, not part of the product
// library: the reference's toy decoder and request loop (reference:
// proj/include/sfi/attention.hpp:46-83, 157-204, proj/include/sfi/
// scheduler.hpp:79-135) with the B200 hot path inside. Built into
// harness/libsfi_toy.so (+ the _sfi_toy Python module) from harness/engine.cpp;
// used by tests/test_engine.py and tests/cpp/test_api.cpp to run the
// reference's acceptance checks (C7-C9) through the device path.
#pragma once

#include <cstdint>
#include <optional>
#include <vector>

#include "sfi/attention.hpp"
#include "sfi/config.hpp"
#include "sfi/scheduler.hpp"
#include "sfi/selector.hpp"

namespace __attribute__((visibility("default"))) sfi {

// ---------------------------------------------------------------------------
// The request loop around the device hot path (engine.cpp).
//
// ToyModel is the reference's small decoder (attention.hpp:46-83,
// model.cpp:36-167; same mt19937_64 / normal_distribution draws, so
// ToyModel::random(spec, seed) holds the reference's weights bit for bit). It
// is the activation source of the end-to-end checks: its
// projections, RoPE, MLP and LM head run on the host in fp64 exactly as the
// reference orders them, while every attention, logit capture, Selector and
// compact rebuild of run_request / run_dense runs through the device path
// (sm_100a kernels over the KvStore's HBM buffers, bf16 KV).
class ToyModel {
 public:
  struct Matrix {  // row-major (out x in)
    int rows = 0, cols = 0;
    std::vector<double> v;
    const double* row(int r) const { return v.data() + static_cast<std::size_t>(r) * cols; }
  };
  struct LayerWeights {
    std::vector<double> ln1, ln2;
    Matrix wq, wk, wv, wo;
    Matrix w_gate, w_up, w_down;
  };
  static ToyModel random(const ModelSpec& spec, std::uint64_t seed);

  const ModelSpec& spec() const { return spec_; }
  const Matrix& embedding() const { return embed_; }
  const LayerWeights& layer(int i) const { return layers_[i]; }
  const std::vector<double>& final_norm() const { return ln_f_; }
  const Matrix& lm_head() const { return lm_head_; }
  const std::vector<double>& lm_bias() const { return lm_bias_; }

 private:
  ModelSpec spec_;
  Matrix embed_;
  std::vector<LayerWeights> layers_;
  std::vector<double> ln_f_;
  Matrix lm_head_;
  std::vector<double> lm_bias_;
};

// attention.hpp:157-182
struct StepOutput {
  std::vector<double> vocab_logits;
  std::optional<std::vector<LogitWindow>> attn_logits;  // slow steps: one window per layer
  std::uint64_t flop_count = 0;
  std::uint64_t kv_read_count = 0;
};
struct CaptureSpec {
  bool window = false;
  std::vector<Pos> allowed;  // J, ascending, one contiguous range (decode / prefill J)
  PoolMode pool = PoolMode::kMean;
};

// attention.hpp:184-204, attention.cpp:249-254
StepOutput dense_attention_step(const ToyModel& model, TokenId token, KvStore& store,
                                const CaptureSpec& capture);
StepOutput sparse_attention_step(const ToyModel& model, TokenId token, KvStore& store,
                                 const std::vector<SupportSet>& support);
std::vector<LogitWindow> prefill_dense(const ToyModel& model, const std::vector<TokenId>& tokens,
                                       KvStore& store, int window_width, const std::vector<Pos>& allowed,
                                       PoolMode pool);
TokenId argmax_token(const std::vector<double>& logits);

// scheduler.hpp:79-135 (StepCause / StepRecord: sfi/scheduler.hpp)
struct RunOptions {
  bool collect_logits = true;
  bool capture_selected = false;
};
struct RequestResult {
  std::vector<TokenId> tokens;
  std::vector<StepRecord> log;
  std::vector<std::vector<double>> step_logits;
  std::uint64_t total_flops = 0;
  std::uint64_t total_kv_reads = 0;
  std::uint64_t dense_equiv_reads = 0;
  std::vector<double> fast_retention;
  std::vector<std::vector<std::vector<std::vector<Pos>>>> selected_per_step;
};
struct DenseResult {
  std::vector<TokenId> tokens;
  std::vector<std::vector<double>> step_logits;
  std::uint64_t total_kv_reads = 0;
  std::uint64_t total_flops = 0;
};
RequestResult run_request(const ToyModel& model, const std::vector<TokenId>& prompt, const CacheLimits& limits,
                          const TriggerConfig& trig, const SelectorConfig& cfg, int max_new,
                          const RunOptions& opts = {});
DenseResult run_dense(const ToyModel& model, const std::vector<TokenId>& prompt, int max_new);

}  // namespace sfi

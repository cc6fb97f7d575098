// sfi_b200.hpp — C++ host API mirroring the reference's operator interface
// (namespace sfi, /root/reference/proj/include/sfi/*.hpp) on top of the C ABI
// in sfi_b200.h. Same type names, field names, defaults and error codes; the
// compute runs on the B200 (no CPU fallback: every hot-path call launches the
// sm_100a kernels and throws sfi_b200::Error on failure).
#pragma once

#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "sfi_b200.h"

namespace __attribute__((visibility("default"))) sfi_b200 {

using Pos = std::int32_t;      // 1-based prefix position (distribution.hpp:23-26)
using TokenId = std::int32_t;

// error.hpp:23-34
enum class ErrorCode {
  kConfig,
  kEmptySupport,
  kSupportMismatch,
  kNonFiniteInput,
  kOverlapViolation,
  kStaleCompact,
  kOutOfRange,
  kBadWeightFile,
  kContextOverflow,
  kIo,
  kCuda,         // B200 additions (status >= 100)
  kUnsupported,
};

class Error : public std::runtime_error {
 public:
  Error(ErrorCode code, const std::string& message) : std::runtime_error(message), code_(code) {}
  ErrorCode code() const noexcept { return code_; }

 private:
  ErrorCode code_;
};

[[noreturn]] void fail(ErrorCode code, const std::string& message);
// Throws the Error matching a non-zero sfi_status, with sfi_last_error().
void check(int status);
const char* error_code_name(ErrorCode code);

// config.hpp:28-76
enum class PoolMode { kMean, kMax };

struct SelectorConfig {
  double alpha = 1.0;
  double gamma = 1.0;
  double beta = 1.0;
  double p_curve = 2.0;
  double eta = 0.5;
  double lambda_clip = 0.02;
  double alpha_soft = 0.5;
  double alpha_cross = 0.35;
  double temperature = 1.0;
  int nms_radius = 2;
  double epsilon = 1e-8;
  int k_budget = 2048;
  PoolMode pool = PoolMode::kMean;
  void validate() const;
  sfi_selector_params to_params() const;
};

struct TriggerConfig {
  std::vector<TokenId> trigger_tokens = {0, 1, 2, 3, 4};
  int t_max = 64;
  int window_decode = 1;
  int window_prefill = 16;
  void validate() const;
  bool is_trigger(TokenId id) const;
};

struct CacheLimits {
  int n_sink = 4;
  int n_recent = 256;
  int k_budget = 2048;
  void validate() const;
};

struct Config {
  SelectorConfig selector;
  TriggerConfig trigger;
  CacheLimits limits;
  void validate() const;
};

Config default_config();

// attention.hpp:31-44
struct ModelSpec {
  int n_layers = 2;
  int n_query_heads = 4;
  int n_kv_heads = 2;
  int head_dim = 16;
  int vocab_size = 256;
  int max_positions = 32768;
  double rope_base = 10000.0;
  int hidden() const { return n_query_heads * head_dim; }
  int group_size() const { return n_query_heads / n_kv_heads; }
  void validate() const;
};

// selector.hpp:31-55
inline constexpr double kMaskedLogit = -1e30;

struct LogitWindow {
  int width = 0;
  std::vector<Pos> allowed;
  std::vector<std::vector<double>> values;  // per KV head, W * |J|
  int heads() const { return static_cast<int>(values.size()); }
  double at(int head, int row, int col) const {
    return values[head][static_cast<std::size_t>(row) * allowed.size() + col];
  }
};

struct CacheStats {
  std::vector<std::vector<double>> key_norms;
  Pos j_min = 0;
  Pos j_max = 0;
  std::vector<double> normalized_pos;
};

CacheStats make_cache_stats(std::vector<std::vector<double>> key_norms,
                            const std::vector<Pos>& allowed, double epsilon);

// Device stage dump of run_selector (SelectorTrace::stages, selector.hpp:66-82).
struct SelectorStages {
  std::vector<std::vector<double>> base;         // z = log(s + eps)
  std::vector<std::vector<double>> after_cross;  // after soft-NMS + cross-head
};

// selector.hpp:121-130 — executed by the sm_100a Selector kernels.
std::vector<Pos> select_top_k(const std::vector<double>& scores, const std::vector<Pos>& allowed,
                              int k);
std::vector<std::vector<Pos>> run_selector(const LogitWindow& w, const CacheStats& stats,
                                           const SelectorConfig& cfg,
                                           SelectorStages* stages = nullptr);

// attention.hpp:82-94
struct SupportSet {
  std::vector<Pos> sink;
  std::vector<std::vector<Pos>> selected;
  Pos recent_start = 1;
  int recent_len = 0;
  int size_for_head(int h) const {
    return static_cast<int>(sink.size() + selected[h].size()) + recent_len;
  }
};

struct KernelStats {
  std::uint64_t flops = 0;
  std::uint64_t reads = 0;
};

// RAII device buffers for one sfi_shape (cudaMalloc, zeroed).
class DeviceCache {
 public:
  explicit DeviceCache(const sfi_shape& shape);
  ~DeviceCache();
  DeviceCache(const DeviceCache&) = delete;
  DeviceCache& operator=(const DeviceCache&) = delete;
  const sfi_shape& shape() const { return shape_; }
  const sfi_cache& cache() const { return cache_; }
  const sfi_sizes& sizes() const { return sizes_; }
  float* logits() const { return logits_; }  // pooled-logit scratch [B][H][Lmax]

 private:
  sfi_shape shape_{};
  sfi_cache cache_{};
  sfi_sizes sizes_{};
  float* logits_ = nullptr;
  std::vector<void*> allocs_;
};

// Device-resident mirror of KvStore (attention.hpp:100-155) for one request
// (batch 1): bf16 paged KV + fp64 key norms in HBM, compact segment + recent
// ring rebuilt on the device. `limits` sizes the ring (n_recent) and the
// compact capacity (n_sink + k_budget).
class KvStore {
 public:
  explicit KvStore(const ModelSpec& spec, const CacheLimits& limits = {}, void* stream = nullptr);

  Pos size() const { return len_; }
  const ModelSpec& spec() const { return spec_; }

  void begin_token();
  void append_layer(int layer, const float* k, const float* v);  // H*d fp32 (rounded to bf16)
  void end_token();
  // Prefill helper: appends `count` tokens for every layer at once.
  // k, v: [n_layers][count][H*d] fp32.
  void append_tokens(int count, const float* k, const float* v);

  std::vector<float> key_row(int layer, Pos pos) const;    // H*d
  std::vector<float> value_row(int layer, Pos pos) const;  // H*d
  double key_norm(int layer, int head, Pos pos) const;

  struct CompactSegment {
    std::vector<Pos> positions;
    std::vector<float> k, v;
  };
  void reorganize(int layer, const std::vector<Pos>& sink,
                  const std::vector<std::vector<Pos>>& selected);
  bool compact_valid(int layer) const { return layers_[layer].valid; }
  bool compact_matches(int layer, const std::vector<Pos>& sink,
                       const std::vector<std::vector<Pos>>& selected) const;
  CompactSegment compact(int layer, int head) const;
  std::pair<Pos, int> recent_tail(int n_recent) const;

  const DeviceCache& device() const { return *dev_; }
  void* stream() const { return stream_; }
  // Syncs the device view of (prefix_len, n_sink_b, recent_len).
  void set_window(int n_sink_b, int recent_len) const;

 private:
  struct LayerState {
    std::vector<std::vector<Pos>> positions;  // merged per head
    bool valid = false;
    int n_sink = 0;
  };
  ModelSpec spec_;
  CacheLimits limits_;
  void* stream_;
  std::unique_ptr<DeviceCache> dev_;
  Pos len_ = 0;
  int pending_layers_ = -1;
  std::vector<LayerState> layers_;
  mutable int cur_nsb_ = -1, cur_rl_ = -1, cur_len_ = -1;
};

// attention.hpp:206-217 — one layer, q [Hq*d] (post-rotary), returns [Hq*d].
std::vector<double> attention_kernel_dense(const KvStore& store, int layer,
                                           const std::vector<double>& q, KernelStats* stats);
std::vector<double> attention_kernel_sparse(const KvStore& store, int layer,
                                            const std::vector<double>& q,
                                            const SupportSet& support, KernelStats* stats);
// Slow-step capture (attention.cpp:367-409 at W = 1): dense attention plus
// the GQA-pooled raw logits over the contiguous allowed range J.
struct DenseCapture {
  std::vector<double> context;              // Hq*d
  LogitWindow window;                       // width 1, per KV head |J|
};
DenseCapture dense_capture(const KvStore& store, int layer, const std::vector<double>& q,
                           const std::vector<Pos>& allowed, PoolMode pool);

// scheduler.hpp:30-76 — host-side decode bookkeeping (integer logic).
struct SparseState {
  int layer = 0;
  std::vector<Pos> sink;
  Pos recent_start = 1;
  int recent_len = 0;
  std::vector<std::vector<Pos>> selected;
  std::vector<Pos> recent() const;
  SupportSet support() const;
};

struct DecodeState {
  int t = 0;
  Pos prefix_len = 0;
  int g = 1;
  int steps_since_slow = 0;
  TokenId last_token = -1;
  std::vector<SparseState> per_layer;
};

DecodeState init_decode_state(Pos prompt_len, int n_layers, int n_kv_heads,
                              const CacheLimits& limits);
std::vector<Pos> compute_allowed(const SparseState& state, Pos prefix_len);
int next_step_type(const DecodeState& state, const TriggerConfig& trig);
void fast_step_update(DecodeState& state, const CacheLimits& limits);
void slow_step_update(DecodeState& state,
                      const std::vector<std::vector<std::vector<Pos>>>& selected_per_layer,
                      const CacheLimits& limits);
double flop_model(double prefix_len, double support, double slow_fraction);

}  // namespace sfi_b200

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
#include <optional>
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
  int ff_dim() const { return 2 * hidden(); }
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
  const CacheLimits& limits() const { return limits_; }
  // Syncs the device view of (prefix_len, n_sink_b, recent_len); `len` < 0
  // means size(). A step attends to the token it is appending (attention.cpp:
  // 354-360), so the request loop passes size() + 1 while a token is open.
  void set_window(int n_sink_b, int recent_len, Pos len = -1) const;
  // Cached fp64 key norms of positions [first, first + count) of one head.
  std::vector<double> key_norms(int layer, int head, Pos first, int count) const;
  // Layers of the open token appended so far (-1: no token open).
  int pending_layers() const { return pending_layers_; }

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

// scheduler.hpp:79-135
enum class StepCause { kInitial, kTrigger, kForced, kNone };
struct StepRecord {
  int t = 0;
  bool slow = false;
  StepCause cause = StepCause::kNone;
  int support_size = 0;
  int allowed_size = 0;
  Pos prefix_len = 0;
};
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

}  // namespace sfi_b200

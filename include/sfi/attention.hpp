// sfi/attention.hpp — KV storage and the attention operators (reference:
// proj/include/sfi/attention.hpp:31-44, 82-155, 206-217). Same ModelSpec,
// SupportSet, KernelStats, KvStore interface and kernel entry points; the
// store lives in HBM (bf16 paged K/V, fp64 key norms, compact segment + recent
// ring per layer) and every operator launches the sm_100a kernels through the
// C ABI (sfi_b200.h). The toy decoder (ToyModel, dense/sparse_attention_step,
// prefill_dense) is not part of this library: it is the end-to-end test
// harness (harness/sfi_toy.hpp, libsfi_toy.so).
//
// Contract differences from the fp32 reference store, all inherent to bf16 KV:
// append_layer rounds k/v to bf16 (round-to-nearest-even), so key_at/value_at
// and the compact segment return the rounded values; key norms are computed
// from the stored (rounded) keys in the reference's c-order fp64 sum.
#pragma once

#include <cstdint>
#include <memory>
#include <utility>
#include <vector>

#include "sfi/config.hpp"
#include "sfi/distribution.hpp"
#include "sfi/selector.hpp"
#include "sfi_b200.h"

namespace __attribute__((visibility("default"))) sfi {

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

struct SupportSet {
  std::vector<Pos> sink;
  std::vector<std::vector<Pos>> selected;  // per KV head
  Pos recent_start = 1;
  int recent_len = 0;

  int size_for_head(int h) const { return static_cast<int>(sink.size() + selected[h].size()) + recent_len; }
};

struct KernelStats {
  std::uint64_t flops = 0;
  std::uint64_t reads = 0;
};

// ---- B200: RAII device buffers of one sfi_shape (cudaMalloc, zeroed) ----
class DeviceCache {
 public:
  explicit DeviceCache(const sfi_shape& shape);
  // A view over borrowed paged storage (k_cache, v_cache, key_norms of one
  // layer of another cache, shape.n_layers == 1) with its own compact / ring /
  // selection / length / workspace buffers: a second compact segment over the
  // same KV rows (KvStore's general supports).
  DeviceCache(const sfi_shape& shape, void* k_cache, void* v_cache, double* key_norms);
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

class KvStore {
 public:
  // The reference constructor: default CacheLimits size the recent ring (256
  // rows) and the initial compact capacity (n_sink + k_budget rows per head,
  // grown on demand by reorganize).
  explicit KvStore(const ModelSpec& spec);
  // B200: explicit ring / compact sizing and the CUDA stream the store's
  // operators are ordered on (nullptr = legacy default stream).
  KvStore(const ModelSpec& spec, const CacheLimits& limits, void* stream = nullptr);
  ~KvStore();
  KvStore(const KvStore&) = delete;
  KvStore& operator=(const KvStore&) = delete;

  Pos size() const { return len_; }
  const ModelSpec& spec() const { return spec_; }

  void begin_token();
  void append_layer(int layer, const float* k, const float* v);  // H*d each
  void end_token();

  const float* key_at(int layer, Pos pos) const;    // H*d floats, valid until the next append / reorganize
  const float* value_at(int layer, Pos pos) const;  // H*d floats
  double key_norm(int layer, int head, Pos pos) const;

  struct CompactSegment {
    std::vector<Pos> positions;  // ascending
    std::vector<float> k, v;     // packed, count * head_dim each
  };

  void reorganize(int layer, const std::vector<Pos>& sink, const std::vector<std::vector<Pos>>& selected);
  bool compact_valid(int layer) const { return layers_[layer].valid; }
  bool compact_matches(int layer, const std::vector<Pos>& sink,
                       const std::vector<std::vector<Pos>>& selected) const;
  const CompactSegment& compact(int layer, int head) const;
  std::pair<Pos, int> recent_tail(int n_recent) const;

  void set_access_trace(bool on) { trace_on_ = on; }
  struct CompactAccess {
    int layer;
    int head;
    int slot;
  };
  std::vector<CompactAccess>& access_trace() { return trace_; }
  void record_compact_access(int layer, int head, int slot) const;

  // ---- B200 extensions ----
  // Prefill helper: `count` tokens for every layer at once; k, v: [n_layers][count][H*d].
  void append_tokens(int count, const float* k, const float* v);
  std::vector<float> key_row(int layer, Pos pos) const;    // copy of key_at's H*d values
  std::vector<float> value_row(int layer, Pos pos) const;
  const DeviceCache& device() const { return *dev_; }
  void* stream() const { return stream_; }
  const CacheLimits& limits() const { return limits_; }
  // Device view of (prefix_len, n_sink_b, recent_len); len < 0 means size().
  void set_window(int n_sink_b, int recent_len, Pos len = -1) const;
  // Cached fp64 key norms of positions [first, first + count) of one head.
  std::vector<double> key_norms(int layer, int head, Pos first, int count) const;
  int pending_layers() const { return pending_layers_; }
  // Rows of the compact segment of `layer` (sink + selected merged, ascending).
  int compact_rows(int layer, int head) const;
  bool trace_on() const { return trace_on_; }

 private:
  struct LayerState {
    std::vector<std::vector<Pos>> positions;  // merged per head
    bool valid = false;
    // general layout (a sink other than {1..m <= n_sink}, or more rows than the
    // store's compact capacity): merged rows gathered into a view of this layer
    std::unique_ptr<DeviceCache> view;
  };
  struct HostMirror {  // lazily filled fp32 copies behind key_at / value_at / compact
    std::vector<float> k, v;   // [len][H*d]
    Pos rows = 0;
    std::vector<CompactSegment> compact;
    std::vector<bool> compact_fresh;
  };
  void sync_host_rows(int layer) const;
  friend std::vector<double> attention_kernel_sparse(const KvStore&, int, const std::vector<double>&,
                                                     const SupportSet&, KernelStats*);

  ModelSpec spec_;
  CacheLimits limits_;
  void* stream_;
  std::unique_ptr<DeviceCache> dev_;
  Pos len_ = 0;
  int pending_layers_ = -1;
  std::vector<LayerState> layers_;
  mutable std::vector<HostMirror> mirror_;
  mutable int cur_nsb_ = -1, cur_rl_ = -1, cur_len_ = -1;
  mutable std::unique_ptr<DeviceCache> support_view_;  // per-call general supports (attention_kernel_sparse)
  bool trace_on_ = false;
  mutable std::vector<CompactAccess> trace_;
};

std::vector<double> attention_kernel_dense(const KvStore& store, int layer, const std::vector<double>& q,
                                           KernelStats* stats);
std::vector<double> attention_kernel_sparse(const KvStore& store, int layer, const std::vector<double>& q,
                                            const SupportSet& support, KernelStats* stats);

// ---- B200: slow-step capture as an operator (attention.cpp:367-409 at W = 1):
// dense attention plus the GQA-pooled raw logits over an ascending allowed list.
struct DenseCapture {
  std::vector<double> context;  // Hq*d
  LogitWindow window;           // width 1, per KV head |J|
};
DenseCapture dense_capture(const KvStore& store, int layer, const std::vector<double>& q,
                           const std::vector<Pos>& allowed, PoolMode pool);

// ---- B200: C ABI status -> sfi::Error (message from sfi_last_error) ----
void check(int status);
sfi_selector_params to_params(const SelectorConfig& cfg);

}  // namespace sfi

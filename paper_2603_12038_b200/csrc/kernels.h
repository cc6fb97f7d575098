// kernels.h — internal launch interface between the C-ABI (capi.cu) and the
// kernel translation units. Not part of the public boundary.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <utility>

#include <cuda_bf16.h>

#include "sfi_b200.h"

namespace sfi_impl {

// Launch with programmatic stream serialization (PDL) unless SFI_PDL=0.
bool pdl_enabled();
// Thread-safe, once per (kernel, size): raise the kernel's dynamic shared
// memory cap to at least `smem` bytes (and allow non-portable cluster sizes).
cudaError_t ensure_kernel_attrs(const void* fn, int smem, bool nonportable_cluster = false);
template <typename... KArgs, typename... Args>
cudaError_t launch_k(void (*fn)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                     Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, fn, std::forward<Args>(args)...);
}

constexpr int kMaxCtas = 1024;  // stream-K decode grid cap (2 partial slots per CTA)

struct DecodeParams {
  const float* q;      // [B][Hq][D]
  float* out;          // [B][Hq][D]
  float* lse;          // [B][Hq] natural-log sum-exp (partial mode for sequence shards) or null
  float* logits;       // [B][H][Lmax] pooled logits over J (dense only) or null
  int pool;
  int layer, B, H, Hq, Lmax, crows, R;
  int sparse;
  const int32_t* prefix_len;
  const int32_t* n_sink_b;
  const int32_t* recent_len;
  const int32_t* n_sel;  // [layers][B][H]
  float* part_o;         // [kMaxCtas][2][8][D]   per-CTA partial O (first / last slice)
  float* part_ml;        // [kMaxCtas][2][2][8]   per-CTA partial (m, l)
  int32_t* counters;     // [B*H], zero between launches
  uint32_t* err;
  float scale_log2;      // log2(e) / sqrt(d)
  float inv_sqrt_d;
  long long* trace;      // debug: per-CTA globaltimer stamps [grid][16] (null = off)
};

// debug / tuning hooks (capi.cu): SFI_DECODE_CTAS overrides the decode grid,
// SFI_DECODE_TRACE=1 records per-CTA timelines readable with sfi_debug_decode_trace.
long long* decode_trace_buffer();

int decode_smem_bytes(int D, int G, int slices);
// stream-K grid: `permille` / 1000 of the 2-CTAs-per-SM capacity, at most one CTA per tile
int decode_grid(int tiles_upper, int num_sms, int permille);
cudaError_t launch_decode(const DecodeParams& p, const CUtensorMap& tmk, const CUtensorMap& tmv,
                          int D, int G, int ctas, cudaStream_t stream);

// fast_decode.cu: fast-step sparse decode, optionally fused with the append
struct FastParams {
  const float* q;                 // [B][Hq][D]
  float* out;                     // [B][Hq][D]
  const __nv_bfloat16* k_new;     // [B][H][D] current token (null: already appended)
  const __nv_bfloat16* v_new;
  __nv_bfloat16* kc;              // paged cache (persist the current token)
  __nv_bfloat16* vc;
  __nv_bfloat16* ck;              // compact cache (ring slot)
  __nv_bfloat16* cv;
  double* norms;
  const int32_t* prefix_len;
  const int32_t* n_sink_b;
  const int32_t* recent_len;
  const int32_t* n_sel;           // [layers][B][H]
  uint32_t* err;
  int layer, B, H, Hq, Lmax, crows, R;
  int prefetch;                   // SFI_FAST_PREFETCH: stream before the PDL wait
  float scale_log2;               // log2(e) / sqrt(d)
  long long* trace;               // debug: per-CTA globaltimer stamps [grid][16] (null = off)
  float* lse;                     // [B][Hq] partial mode (sequence shards): LSE out, empty allowed
  int32_t* steal;                 // [layers][B][H][2] tile-claim / done counters (null: static split)
};
int fast_cluster_size(int slices, int num_sms, int tiles);  // tiles: 64-row tiles of one compact slice
cudaError_t launch_fast_decode(const FastParams& p, const CUtensorMap& tmk, const CUtensorMap& tmv, int D,
                               int G, int C, cudaStream_t stream);

// cache_ops.cu
cudaError_t launch_step_advance(const sfi_shape& s, const sfi_cache& c, cudaStream_t st);
cudaError_t launch_set_recent_rule(const sfi_shape& s, const sfi_cache& c, cudaStream_t st);
cudaError_t launch_append(const sfi_shape& s, const sfi_cache& c, int layer, int count,
                          const void* k, const void* v, int advance_ring_only_current,
                          cudaStream_t st);
cudaError_t launch_compact_build(const sfi_shape& s, const sfi_cache& c, int layer,
                                 int rebuild_ring, cudaStream_t st);
cudaError_t launch_fill_synthetic(const sfi_shape& s, const sfi_cache& c, uint64_t seed, int len,
                                  cudaStream_t st);

// selector.cu
struct SelectorScratch {
  double* a;      // [B*H][Lmax]  p -> weights -> f -> z_base
  double* b;      // [B*H][Lmax]  w -> r -> z_adj
  double* c;      // [B*H][Lmax]  prior weights w (two-pass decode Selector)
  double* stats;  // [B*H][ceil(Lmax / 512)][6] chunk statistics, then [B*H][chunks + 2] coefficients
  void* bt = nullptr;  // long-row top-k buffers (sel_bt_*)
};
constexpr int kTopkCtaMaxPositions = 48 * 1024;  // rows up to this length: the single-CTA top-k
// phases: 1 = fuse (z_base into scr.a), 2 = refine + top-k; z_all != null:
// head-sharded finish over the all-gathered z_base of n_shards shards
cudaError_t launch_selector(const sfi_shape& s, const sfi_cache& c, int layer, const float* logits,
                            const sfi_selector_params& prm, const SelectorScratch& scr,
                            cudaStream_t st, int* launches, int phases = 3,
                            const double* z_all = nullptr, int n_shards = 1, int shard = 0, int W = 1);

cudaError_t launch_selector_explicit(int H, int W, int n, int K, const double* logits,
                                     const double* norms, const int32_t* allowed,
                                     const sfi_selector_params& prm, double* sa, double* sb,
                                     int32_t* sel, int32_t* n_sel, uint32_t* err, cudaStream_t st,
                                     int* launches);
cudaError_t launch_floor(int n, int grid, cudaStream_t st);
// K1 on tcgen05 (dense, D = 128, G in {4, 8, 16}): tensor maps with 64 x 128 boxes
cudaError_t launch_decode_tc(const DecodeParams& p, const CUtensorMap& tmk128, const CUtensorMap& tmv128, int G,
                             int stages, int ctas, cudaStream_t stream);
int decode_tc_tiles_upper(int max_positions);
cudaError_t launch_selector_stage(int stage, int H, int W, int n, const double* a, const double* b,
                                  const sfi_selector_params& prm, double* out, double* out2, int32_t* head_err,
                                  cudaStream_t st);
cudaError_t launch_topk_explicit(int rows, int n, int K, const double* scores, const int32_t* allowed,
                                 int32_t* sel, int32_t* n_sel, cudaStream_t st, int* launches);

// sequence sharding
cudaError_t launch_seq_lengths(const sfi_shape& s, const sfi_cache& c, int32_t* g_prefix, const int32_t* g_nsink,
                               int32_t* g_recent, int advance, int base, int is_last, int32_t* j_off,
                               int32_t* n_glob, cudaStream_t st);
constexpr int kMaxPeers = 64;
cudaError_t launch_peer_publish(int32_t* flag, cudaStream_t st);
cudaError_t launch_peer_gather(int n_parts, long long words, const uint32_t* const* src, const int32_t* const* flags,
                               const int32_t* my_flag, uint32_t* dst, cudaStream_t st);
cudaError_t launch_peer_merge(int n_parts, int rows, int D, const float* const* o_ptrs, const float* const* lse_ptrs,
                              const int32_t* const* flags, const int32_t* my_flag, float* out, cudaStream_t st);
cudaError_t launch_merge_partials(int n_parts, int rows, int D, const float* o_parts, const float* lse_parts,
                                  float* out, cudaStream_t st);
cudaError_t launch_seq_selector_stats(const sfi_shape& s, const sfi_cache& c, int layer, const float* logits,
                                      const sfi_selector_params& prm, const SelectorScratch& scr,
                                      const int32_t* j_off, const int32_t* n_glob, int phase, double* row_stats,
                                      const double* stats_all, int n_shards, double* edges, cudaStream_t st);
cudaError_t launch_seq_selector_finish(const sfi_shape& s, const sfi_cache& c, int layer,
                                       const sfi_selector_params& prm, const SelectorScratch& scr,
                                       const int32_t* j_off, const int32_t* n_glob, const double* edges_all,
                                       int n_shards, int pos_base, double* cand_score, int32_t* cand_pos,
                                       cudaStream_t st, int* launches);
size_t seq_pick_scratch_bytes(const sfi_shape& s, int n_shards);
cudaError_t launch_seq_selector_pick(const sfi_shape& s, const sfi_cache& c, int layer, int n_shards,
                                     const double* cand_score_all, const int32_t* cand_pos_all, int pos_base,
                                     int pos_end, void* scratch, cudaStream_t st, int* launches);

// capture.cu: prefill tail-window capture
struct CaptureParams {
  const float* q;              // [B][W][Hq][D]
  const int32_t* q_pos;        // [B][W] 1-based positions of the window rows
  const __nv_bfloat16* k_cache;
  float* out;                  // [B][H][W][Lmax], entry (b, h, w, p - j_min)
  const int32_t* prefix_len;
  const int32_t* n_sink_b;
  const int32_t* recent_len;
  int layer, B, H, Hq, Lmax, W, pool;
  float inv_sqrt_d;
};
cudaError_t launch_capture(const CaptureParams& p, int D, cudaStream_t st);

// workspace carve-up (capi.cu)
struct Workspace {
  float* part_o;
  float* part_ml;
  int32_t* counters;
  SelectorScratch sel;
  int32_t* steal;  // [layers][B][H][2] fast-decode tile-claim counters (zero at rest)
};
size_t workspace_bytes(const sfi_shape& s);
Workspace carve_workspace(const sfi_shape& s, void* base);

}  // namespace sfi_impl

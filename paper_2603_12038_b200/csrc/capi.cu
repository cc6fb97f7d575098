// capi.cu — the extern "C" boundary (include/sfi_b200.h): argument
// validation, TMA descriptor encoding, workspace carve-up, kernel launches,
// status codes and a thread-local error message. No exceptions cross it.
#include <cuda.h>
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include "kernels.h"
#include "sfi_b200.h"

namespace {

thread_local std::string g_err;
thread_local int32_t g_launches = 0;
int g_trace_ctas = 0;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

int cuda_fail(cudaError_t e, const char* where) {
  return fail(SFI_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

#define SFI_CUDA(call, where)                      \
  do {                                             \
    cudaError_t e_ = (call);                       \
    if (e_ != cudaSuccess) return cuda_fail(e_, where); \
  } while (0)

size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

int group_of(const sfi_shape& s) { return s.n_q_heads / s.n_kv_heads; }
int compact_rows(const sfi_shape& s) { return s.n_recent + s.n_sink + s.k_budget; }

int validate(const sfi_shape* s) {
  if (!s) return fail(SFI_ERR_INVALID_ARGUMENT, "shape is null");
  if (s->n_layers < 1 || s->batch < 1 || s->n_kv_heads < 1 || s->n_q_heads < 1)
    return fail(SFI_ERR_CONFIG, "shape: n_layers, batch and head counts must be >= 1");
  if (s->n_q_heads % s->n_kv_heads != 0)
    return fail(SFI_ERR_CONFIG, "shape: n_q_heads must be a multiple of n_kv_heads");
  const int G = group_of(*s);
  if (G != 1 && G != 2 && G != 4 && G != 8 && G != 16)
    return fail(SFI_ERR_UNSUPPORTED, "shape: GQA group size must be 1, 2, 4, 8 or 16");
  if (s->head_dim != 64 && s->head_dim != 128)
    return fail(SFI_ERR_UNSUPPORTED, "shape: head_dim must be 64 or 128");
  if (s->n_kv_heads > 16) return fail(SFI_ERR_UNSUPPORTED, "shape: at most 16 KV heads");
  if ((long long)s->batch * s->n_kv_heads > 4096)
    return fail(SFI_ERR_UNSUPPORTED, "shape: at most 4096 (request, KV head) slices");
  if (s->max_positions < 1) return fail(SFI_ERR_CONFIG, "shape: max_positions must be >= 1");
  if (s->n_sink < 0 || s->k_budget < 0 || s->n_recent < 1)
    return fail(SFI_ERR_CONFIG, "shape: n_sink >= 0, k_budget >= 0, n_recent >= 1 required");
  const double rows = double(s->n_layers) * s->batch * s->n_kv_heads *
                      std::max(s->max_positions, compact_rows(*s));
  if (rows >= 2147483647.0)
    return fail(SFI_ERR_UNSUPPORTED, "shape: more than 2^31 cache rows (TMA coordinate range)");
  return SFI_OK;
}

int check_layer(const sfi_shape* s, int layer) {
  if (layer < 0 || layer >= s->n_layers) return fail(SFI_ERR_OUT_OF_RANGE, "layer out of range");
  return SFI_OK;
}

int check_cache(const sfi_shape* s, const sfi_cache* c) {
  if (!c || !c->k_cache || !c->v_cache || !c->key_norms || !c->ck || !c->cv || !c->sel ||
      !c->n_sel || !c->prefix_len || !c->n_sink_b || !c->recent_len || !c->error_flags || !c->workspace)
    return fail(SFI_ERR_INVALID_ARGUMENT, "cache: null buffer");
  if (c->workspace_bytes < sfi_impl::workspace_bytes(*s))
    return fail(SFI_ERR_INVALID_ARGUMENT, "cache: workspace too small");
  return SFI_OK;
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                              CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encode_fn() {
  static EncodeFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(p);
  });
  return fn;
}

// 2D bf16 view [rows][D] with 64-column x box_rows boxes, 128-byte swizzle.
int make_tmap(CUtensorMap* m, void* base, uint64_t rows, int D, uint32_t box_rows = 64) {
  EncodeFn fn = encode_fn();
  if (!fn) return fail(SFI_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  const cuuint64_t dims[2] = {(cuuint64_t)D, rows};
  const cuuint64_t strides[1] = {(cuuint64_t)D * 2};
  const cuuint32_t box[2] = {64, box_rows};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(SFI_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
  return SFI_OK;
}

int num_sms() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

int decode_common(const sfi_shape* s, const sfi_cache* c, int layer, const float* q, float* out,
                  float* logits, int pool, bool sparse, void* stream, float* lse = nullptr, int flags = 0) {
  g_launches = 0;
  int rc = validate(s);
  if (rc) return rc;
  if ((rc = check_cache(s, c)) || (rc = check_layer(s, layer))) return rc;
  if (!q || !out) return fail(SFI_ERR_INVALID_ARGUMENT, "decode: q/out null");
  if (pool != SFI_POOL_MEAN && pool != SFI_POOL_MAX) return fail(SFI_ERR_CONFIG, "decode: bad pool mode");
  const int D = s->head_dim;
  const uint64_t slices = (uint64_t)s->n_layers * s->batch * s->n_kv_heads;
  const uint64_t rows_per = sparse ? (uint64_t)compact_rows(*s) : (uint64_t)s->max_positions;
  CUtensorMap tk, tv;
  if ((rc = make_tmap(&tk, sparse ? c->ck : c->k_cache, slices * rows_per, D))) return rc;
  if ((rc = make_tmap(&tv, sparse ? c->cv : c->v_cache, slices * rows_per, D))) return rc;
  sfi_impl::Workspace ws = sfi_impl::carve_workspace(*s, c->workspace);
  sfi_impl::DecodeParams p;
  p.q = q;
  p.out = out;
  p.lse = lse;
  p.logits = sparse ? nullptr : logits;
  p.pool = pool;
  p.layer = layer;
  p.B = s->batch;
  p.H = s->n_kv_heads;
  p.Hq = s->n_q_heads;
  p.Lmax = s->max_positions;
  p.crows = compact_rows(*s);
  p.R = s->n_recent;
  p.sparse = sparse ? 1 : 0;
  p.prefix_len = c->prefix_len;
  p.n_sink_b = c->n_sink_b;
  p.recent_len = c->recent_len;
  p.n_sel = c->n_sel;
  p.part_o = ws.part_o;
  p.part_ml = ws.part_ml;
  p.counters = ws.counters;
  p.err = c->error_flags;
  p.inv_sqrt_d = (float)(1.0 / std::sqrt((double)D));
  p.scale_log2 = (float)(1.4426950408889634 / std::sqrt((double)D));
  const int per_slice = sparse ? (s->n_recent + 63) / 64 + 1 + (s->n_sink + s->k_budget + 63) / 64
                              : (s->max_positions + 63) / 64;
  // 7/8 of the 2-CTAs-per-SM slots measures fastest alone (fewer in-flight
  // streams per HBM channel); SFI_DENSE_SHARE_SM keeps 65% (192 CTAs on 148
  // SMs, the measured optimum of the asynchronous slow-step pipeline) and
  // leaves the rest to the Selector kernels running beside it
  static const int env_share = [] {
    const char* e = std::getenv("SFI_DENSE_SHARE_PERMILLE");
    return e ? std::atoi(e) : 0;
  }();
  // measured optimum of the async slow step per group size (profiles/r02/share_sweep.txt,
  // 3 repeats each): G = 4 (C2) 67.5% of the 2-CTA slots (8.23 vs 8.37 ms at 65%),
  // G = 8 (C3) 75% (27.9 vs 30.4 ms), G = 2 (C1) 50% (1.02 vs 1.04 ms); G = 16 (C4) takes
  // the tcgen05 kernel on 77.5% of the SMs
  const int Gq = s->n_q_heads / s->n_kv_heads;
  const int share = (env_share > 0 && env_share <= 1000) ? env_share
                    : (Gq >= 16 ? 1000 : Gq >= 8 ? 750 : Gq >= 4 ? 675 : 500);
  int ctas = sfi_impl::decode_grid(per_slice * s->batch * s->n_kv_heads, num_sms(),
                                   (flags & SFI_DENSE_SHARE_SM) ? share : 875);
  static const int env_ctas = [] {
    const char* e = std::getenv("SFI_DECODE_CTAS");
    return e ? std::atoi(e) : 0;
  }();
  if (env_ctas > 0) ctas = std::min(env_ctas, sfi_impl::kMaxCtas);
  p.trace = nullptr;
  static const bool env_trace = std::getenv("SFI_DECODE_TRACE") != nullptr;
  const bool trace_on = env_trace;
  if (env_trace) {
    p.trace = sfi_impl::decode_trace_buffer();
    if (!p.trace) return fail(SFI_ERR_CUDA, "trace buffer");
    SFI_CUDA(cudaMemsetAsync(p.trace, 0, sizeof(long long) * 16 * sfi_impl::kMaxCtas, (cudaStream_t)stream),
             "trace");
    g_trace_ctas = ctas;
  }
  // K1 on tcgen05: dense, D = 128, G in {4, 8, 16}; one CTA per SM
  static const int env_tc = [] {  // default on; SFI_DENSE_TC=0 selects the mma.sync kernel
    const char* e = std::getenv("SFI_DENSE_TC");
    return e ? std::atoi(e) : 1;
  }();
  const int G = group_of(*s);
  // default: the tcgen05 kernel, except beside the Selector at G <= 8 (SFI_DENSE_SHARE_SM),
  // where the mma.sync kernel's 2 CTAs per SM on 65% of the slots overlap the Selector
  // chain better (C2 async slow step 8.33 vs 8.49 ms per step, measured)
  static const int env_tc_share_g = [] {  // smallest group that takes tcgen05 beside the Selector
    const char* e = std::getenv("SFI_DENSE_TC_SHARE_G");
    return e ? std::atoi(e) : 16;
  }();
  const bool share_flag = (flags & SFI_DENSE_SHARE_SM) != 0;
  const bool want_tc = (flags & SFI_DENSE_TC)    ? true
                       : (flags & SFI_DENSE_MMA) ? false
                                                 : env_tc > 0 && (!share_flag || group_of(*s) >= env_tc_share_g);
  if (!sparse && D == 128 && (G == 4 || G == 8 || G == 16) && want_tc) {
    CUtensorMap tk2, tv2;
    if ((rc = make_tmap(&tk2, c->k_cache, slices * rows_per, D, 128))) return rc;
    if ((rc = make_tmap(&tv2, c->v_cache, slices * rows_per, D, 128))) return rc;
    // alone: 3 stages (192 KB) on every SM. Beside the Selector (SFI_DENSE_SHARE_SM):
    // SFI_DENSE_TC_SHARE_PERMILLE of the SMs with SFI_DENSE_TC_SHARE_STAGES stages
    // (default 3; 2 stages, ~150 KB, let Selector CTAs co-reside but measured slower)
    static const int env_tc_share = [] {  // C4: 775 permille 13.8 vs 14.9 ms per slow step on every SM
      const char* e = std::getenv("SFI_DENSE_TC_SHARE_PERMILLE");
      return e ? std::atoi(e) : 775;
    }();
    static const int env_tc_share_stages = [] {  // C4: 3 stages 14.5 vs 2 stages 15.4 ms per slow step
      const char* e = std::getenv("SFI_DENSE_TC_SHARE_STAGES");
      return e ? std::atoi(e) : 3;
    }();
    const bool share_mode = (flags & SFI_DENSE_SHARE_SM) != 0;
    const int share_tc = share_mode ? env_tc_share : 1000;
    const int stages = share_mode ? (env_tc_share_stages == 3 ? 3 : 2) : 3;
    int tc_ctas = std::max(1, std::min(num_sms() * share_tc / 1000,
                                       sfi_impl::decode_tc_tiles_upper(s->max_positions) * s->batch * s->n_kv_heads));
    if (env_ctas > 0) tc_ctas = std::min(env_ctas, num_sms());
    if (trace_on) g_trace_ctas = tc_ctas;
    SFI_CUDA(sfi_impl::launch_decode_tc(p, tk2, tv2, G, stages, tc_ctas, (cudaStream_t)stream),
             "sfi_dense_decode (tcgen05)");
    g_launches = 1;
    return SFI_OK;
  }
  SFI_CUDA(sfi_impl::launch_decode(p, tk, tv, D, G, ctas, (cudaStream_t)stream),
           sparse ? "sfi_sparse_decode" : "sfi_dense_decode");
  g_launches = 1;
  return SFI_OK;
}

constexpr int kLayerTraceMax = 128;
long long* layer_trace_buffer() {
  static long long* buf = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    if (cudaMalloc(&buf, sizeof(long long) * 16 * sfi_impl::kMaxCtas * kLayerTraceMax) != cudaSuccess) buf = nullptr;
    else cudaMemset(buf, 0, sizeof(long long) * 16 * sfi_impl::kMaxCtas * kLayerTraceMax);
  });
  return buf;
}

// Fast step, one layer: sparse decode over the compact cache, fused with the
// current token's append when k_new / v_new are given (fast_decode.cu).
int fast_common(const sfi_shape* s, const sfi_cache* c, int layer, const float* q, const void* k_new,
                const void* v_new, float* out, int flags, void* stream, float* lse = nullptr) {
  g_launches = 0;
  int rc = validate(s);
  if (rc) return rc;
  if ((rc = check_cache(s, c)) || (rc = check_layer(s, layer))) return rc;
  if (!q || !out) return fail(SFI_ERR_INVALID_ARGUMENT, "decode: q/out null");
  if ((k_new == nullptr) != (v_new == nullptr)) return fail(SFI_ERR_INVALID_ARGUMENT, "fast_decode: k/v null");
  if (flags & ~SFI_FAST_PREFETCH) return fail(SFI_ERR_INVALID_ARGUMENT, "fast_decode: unknown flags");
  const int D = s->head_dim;
  const uint64_t slices = (uint64_t)s->n_layers * s->batch * s->n_kv_heads;
  CUtensorMap tk, tv;
  if ((rc = make_tmap(&tk, c->ck, slices * compact_rows(*s), D))) return rc;
  if ((rc = make_tmap(&tv, c->cv, slices * compact_rows(*s), D))) return rc;
  sfi_impl::FastParams p;
  p.q = q;
  p.out = out;
  p.k_new = static_cast<const __nv_bfloat16*>(k_new);
  p.v_new = static_cast<const __nv_bfloat16*>(v_new);
  p.kc = static_cast<__nv_bfloat16*>(c->k_cache);
  p.vc = static_cast<__nv_bfloat16*>(c->v_cache);
  p.ck = static_cast<__nv_bfloat16*>(c->ck);
  p.cv = static_cast<__nv_bfloat16*>(c->cv);
  p.norms = c->key_norms;
  p.prefix_len = c->prefix_len;
  p.n_sink_b = c->n_sink_b;
  p.recent_len = c->recent_len;
  p.n_sel = c->n_sel;
  p.err = c->error_flags;
  p.layer = layer;
  p.B = s->batch;
  p.H = s->n_kv_heads;
  p.Hq = s->n_q_heads;
  p.Lmax = s->max_positions;
  p.crows = compact_rows(*s);
  p.R = s->n_recent;
  p.prefetch = (flags & SFI_FAST_PREFETCH) ? 1 : 0;
  p.lse = lse;
  p.scale_log2 = (float)(1.4426950408889634 / std::sqrt((double)D));
  static const bool env_steal = [] {
    const char* e = std::getenv("SFI_FAST_STEAL");
    return e && e[0] == '1';
  }();
  p.steal = env_steal ? sfi_impl::carve_workspace(*s, c->workspace).steal : nullptr;
  static const int env_c = [] {
    const char* e = std::getenv("SFI_FAST_CLUSTER");
    return e ? std::atoi(e) : 0;
  }();
  const int fast_tiles = (s->n_recent + 63) / 64 + (s->n_sink + s->k_budget + 63) / 64;
  int C = sfi_impl::fast_cluster_size(s->batch * s->n_kv_heads, num_sms(), fast_tiles);
  if (env_c >= 1 && env_c <= 16) C = env_c;
  p.trace = nullptr;
  static const bool env_trace = std::getenv("SFI_DECODE_TRACE") != nullptr;
  static const bool env_layer_trace = std::getenv("SFI_LAYER_TRACE") != nullptr;
  const int grid = s->batch * s->n_kv_heads * C;
  if (env_layer_trace && grid <= sfi_impl::kMaxCtas && layer < kLayerTraceMax) {
    // per-layer slots, no reset: a graph of one step's launches leaves every
    // layer's CTA timeline behind (sfi_debug_layer_trace)
    long long* buf = layer_trace_buffer();
    if (!buf) return fail(SFI_ERR_CUDA, "layer trace buffer");
    p.trace = buf + (size_t)layer * sfi_impl::kMaxCtas * 16;
    g_trace_ctas = grid;
  } else if (env_trace && grid <= sfi_impl::kMaxCtas) {
    p.trace = sfi_impl::decode_trace_buffer();
    if (!p.trace) return fail(SFI_ERR_CUDA, "trace buffer");
    SFI_CUDA(cudaMemsetAsync(p.trace, 0, sizeof(long long) * 16 * sfi_impl::kMaxCtas, (cudaStream_t)stream),
             "trace");
    g_trace_ctas = grid;
  }
  SFI_CUDA(sfi_impl::launch_fast_decode(p, tk, tv, D, group_of(*s), C, (cudaStream_t)stream),
           k_new ? "sfi_fast_decode" : "sfi_sparse_decode");
  g_launches = 1;
  return SFI_OK;
}

}  // namespace

namespace sfi_impl {

cudaError_t ensure_kernel_attrs(const void* fn, int smem, bool nonportable_cluster) {
  static std::mutex mu;
  static std::unordered_map<const void*, int> caps;  // configured smem cap per kernel
  std::lock_guard<std::mutex> lock(mu);
  auto it = caps.find(fn);
  if (it != caps.end() && it->second >= smem) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e == cudaSuccess && nonportable_cluster)
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  if (e == cudaSuccess) caps[fn] = smem;
  return e;
}

bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("SFI_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

long long* decode_trace_buffer() {
  static long long* buf = nullptr;
  if (!buf && cudaMalloc(&buf, sizeof(long long) * 16 * kMaxCtas) != cudaSuccess) buf = nullptr;
  return buf;
}

// rows of one stream-K partial: 8, or 16 for GQA group 16 (decode.cu part_rows)
static size_t part_rows(const sfi_shape& s) { return group_of(s) > 8 ? 16 : 8; }

// long-row top-k buffers (selector.cu sel_bt_*; the default when |J| can exceed the
// single-CTA top-k, SFI_TOPK_BT=1 for every length): [rows][65536 + 1024] bin and chunk counts, [rows][max_positions] listed
// indices, [rows][8] row state, [rows][64][2] segment counts / offsets
size_t bt_bytes(const sfi_shape& s) {
  const size_t rows = (size_t)s.batch * s.n_kv_heads;
  return rows * (65536 * 4 + (size_t)s.max_positions * 4 + 16 * 4 + 64 * 2 * 4);
}

size_t workspace_bytes(const sfi_shape& s) {
  const size_t slices = (size_t)s.batch * s.n_kv_heads;
  size_t b = 0;
  b += align_up((size_t)kMaxCtas * 2 * part_rows(s) * s.head_dim * sizeof(float));
  b += align_up((size_t)kMaxCtas * 2 * 2 * part_rows(s) * sizeof(float));
  b += align_up(slices * sizeof(int32_t));
  b += 3 * align_up(slices * (size_t)s.max_positions * sizeof(double));
  // two-pass decode Selector: [rows][chunks][6] statistics + [rows][chunks + 2] coefficients
  b += align_up(slices * (size_t)(7 * ((s.max_positions + 511) / 512) + 2) * sizeof(double));
  b += align_up((size_t)s.n_layers * slices * 2 * sizeof(int32_t));  // fast-decode tile-claim counters
  b += align_up(bt_bytes(s));                                          // long-row top-k (C3 / C4)
  return b;
}

Workspace carve_workspace(const sfi_shape& s, void* base) {
  const size_t slices = (size_t)s.batch * s.n_kv_heads;
  uint8_t* p = static_cast<uint8_t*>(base);
  Workspace w;
  w.part_o = reinterpret_cast<float*>(p);
  p += align_up((size_t)kMaxCtas * 2 * part_rows(s) * s.head_dim * sizeof(float));
  w.part_ml = reinterpret_cast<float*>(p);
  p += align_up((size_t)kMaxCtas * 2 * 2 * part_rows(s) * sizeof(float));
  w.counters = reinterpret_cast<int32_t*>(p);
  p += align_up(slices * sizeof(int32_t));
  w.sel.a = reinterpret_cast<double*>(p);
  p += align_up(slices * (size_t)s.max_positions * sizeof(double));
  w.sel.b = reinterpret_cast<double*>(p);
  p += align_up(slices * (size_t)s.max_positions * sizeof(double));
  w.sel.c = reinterpret_cast<double*>(p);
  p += align_up(slices * (size_t)s.max_positions * sizeof(double));
  w.sel.stats = reinterpret_cast<double*>(p);
  p += align_up(slices * (size_t)(7 * ((s.max_positions + 511) / 512) + 2) * sizeof(double));
  w.steal = reinterpret_cast<int32_t*>(p);
  p += align_up((size_t)s.n_layers * slices * 2 * sizeof(int32_t));
  w.sel.bt = bt_bytes(s) ? p : nullptr;
  return w;
}

}  // namespace sfi_impl

extern "C" {

SFI_API const char* sfi_version(void) { return "sfi_b200 0.1 (sm_100a)"; }
SFI_API const char* sfi_last_error(void) { return g_err.c_str(); }
SFI_API int32_t sfi_last_launch_count(void) { return g_launches; }

SFI_API int32_t sfi_debug_layer_trace(int64_t* out, int32_t layers, int32_t max_ctas) {
  long long* buf = layer_trace_buffer();
  if (!buf || !out || layers <= 0 || layers > kLayerTraceMax || max_ctas <= 0) return 0;
  const int n = std::min(max_ctas, sfi_impl::kMaxCtas);
  for (int l = 0; l < layers; ++l)
    if (cudaMemcpy(out + (size_t)l * n * 16, buf + (size_t)l * sfi_impl::kMaxCtas * 16, sizeof(long long) * 16 * n,
                   cudaMemcpyDeviceToHost) != cudaSuccess)
      return 0;
  return g_trace_ctas;
}

SFI_API int32_t sfi_debug_decode_trace(int64_t* out, int32_t max_ctas) {
  long long* buf = sfi_impl::decode_trace_buffer();
  const int n = std::min(max_ctas, g_trace_ctas);
  if (!buf || !out || n <= 0) return 0;
  if (cudaMemcpy(out, buf, sizeof(long long) * 16 * n, cudaMemcpyDeviceToHost) != cudaSuccess) return 0;
  return n;
}

SFI_API int sfi_shape_validate(const sfi_shape* shape) { return validate(shape); }

SFI_API int sfi_buffer_sizes(const sfi_shape* s, sfi_sizes* out) {
  int rc = validate(s);
  if (rc) return rc;
  if (!out) return fail(SFI_ERR_INVALID_ARGUMENT, "sizes: out is null");
  const size_t slices = (size_t)s->n_layers * s->batch * s->n_kv_heads;
  out->kv_cache = slices * s->max_positions * s->head_dim * 2;
  out->key_norms = slices * s->max_positions * sizeof(double);
  out->compact = slices * compact_rows(*s) * s->head_dim * 2;
  out->sel = slices * (size_t)std::max(1, s->k_budget) * sizeof(int32_t);
  out->n_sel = slices * sizeof(int32_t);
  out->per_batch = (size_t)s->batch * sizeof(int32_t);
  out->workspace = sfi_impl::workspace_bytes(*s);
  out->pooled_logits = (size_t)s->batch * s->n_kv_heads * s->max_positions * sizeof(float);
  return SFI_OK;
}

SFI_API void sfi_default_selector_params(sfi_selector_params* o) {
  // SelectorConfig defaults, config.hpp:31-47
  o->alpha = 1.0;
  o->gamma = 1.0;
  o->beta = 1.0;
  o->p_curve = 2.0;
  o->eta = 0.5;
  o->lambda_clip = 0.02;
  o->alpha_soft = 0.5;
  o->alpha_cross = 0.35;
  o->temperature = 1.0;
  o->epsilon = 1e-8;
  o->nms_radius = 2;
  o->pool = SFI_POOL_MEAN;
}

SFI_API void sfi_recent_window(int32_t prefix_len, int32_t n_sink_b, int32_t n_recent,
                               int32_t* recent_start, int32_t* recent_len) {
  int rl = prefix_len - n_sink_b;
  rl = rl < 0 ? 0 : (rl > n_recent ? n_recent : rl);
  if (recent_len) *recent_len = rl;
  if (recent_start) *recent_start = prefix_len - rl + 1;
}

SFI_API int sfi_set_lengths(const sfi_shape* s, const sfi_cache* c, const int32_t* prefix_len_host,
                            const int32_t* n_sink_host, const int32_t* recent_len_host, void* stream) {
  g_launches = 0;
  int rc = validate(s);
  if (rc || (rc = check_cache(s, c))) return rc;
  if (!prefix_len_host || !n_sink_host) return fail(SFI_ERR_INVALID_ARGUMENT, "set_lengths: null argument");
  for (int b = 0; b < s->batch; ++b) {
    if (prefix_len_host[b] < 0 || prefix_len_host[b] > s->max_positions)
      return fail(SFI_ERR_CONTEXT_OVERFLOW, "set_lengths: prefix length exceeds max_positions");
    // n_sink_b <= n_sink and recent_len <= n_recent are required by the compact
    // layout (checked on the device by sfi_compact_build / sfi_sparse_decode);
    // a dense capture may use any window inside [0, L].
    if (n_sink_host[b] < 0 || n_sink_host[b] > prefix_len_host[b])
      return fail(SFI_ERR_CONFIG, "set_lengths: n_sink_b must be in [0, L]");
    if (recent_len_host && (recent_len_host[b] < 0 || recent_len_host[b] > prefix_len_host[b]))
      return fail(SFI_ERR_OUT_OF_RANGE, "set_lengths: recent_len must be in [0, L]");
  }
  cudaStream_t st = (cudaStream_t)stream;
  const size_t nb = (size_t)s->batch * sizeof(int32_t);
  SFI_CUDA(cudaMemcpyAsync(c->prefix_len, prefix_len_host, nb, cudaMemcpyHostToDevice, st), "set_lengths");
  SFI_CUDA(cudaMemcpyAsync(c->n_sink_b, n_sink_host, nb, cudaMemcpyHostToDevice, st), "set_lengths");
  if (recent_len_host) {
    SFI_CUDA(cudaMemcpyAsync(c->recent_len, recent_len_host, nb, cudaMemcpyHostToDevice, st), "set_lengths");
  } else {
    SFI_CUDA(sfi_impl::launch_set_recent_rule(*s, *c, st), "set_lengths");
    g_launches = 1;
  }
  SFI_CUDA(cudaStreamSynchronize(st), "set_lengths");
  return SFI_OK;
}

SFI_API int sfi_step_advance(const sfi_shape* s, const sfi_cache* c, void* stream) {
  g_launches = 0;
  int rc = validate(s);
  if (rc || (rc = check_cache(s, c))) return rc;
  SFI_CUDA(sfi_impl::launch_step_advance(*s, *c, (cudaStream_t)stream), "sfi_step_advance");
  g_launches = 1;
  return SFI_OK;
}

SFI_API int sfi_ring_append(const sfi_shape* s, const sfi_cache* c, int32_t layer, const void* k_new,
                            const void* v_new, void* stream) {
  g_launches = 0;
  int rc = validate(s);
  if (rc || (rc = check_cache(s, c)) || (rc = check_layer(s, layer))) return rc;
  if (!k_new || !v_new) return fail(SFI_ERR_INVALID_ARGUMENT, "ring_append: k/v null");
  SFI_CUDA(sfi_impl::launch_append(*s, *c, layer, 1, k_new, v_new, 0, (cudaStream_t)stream),
           "sfi_ring_append");
  g_launches = 1;
  return SFI_OK;
}

SFI_API int sfi_append_block(const sfi_shape* s, const sfi_cache* c, int32_t layer, int32_t count,
                             const void* k, const void* v, void* stream) {
  g_launches = 0;
  int rc = validate(s);
  if (rc || (rc = check_cache(s, c)) || (rc = check_layer(s, layer))) return rc;
  if (count < 0) return fail(SFI_ERR_OUT_OF_RANGE, "append_block: negative count");
  if (count == 0) return SFI_OK;
  if (!k || !v) return fail(SFI_ERR_INVALID_ARGUMENT, "append_block: k/v null");
  SFI_CUDA(sfi_impl::launch_append(*s, *c, layer, count, k, v, 1, (cudaStream_t)stream),
           "sfi_append_block");
  g_launches = 1;
  return SFI_OK;
}

SFI_API int sfi_dense_decode(const sfi_shape* s, const sfi_cache* c, int32_t layer, const float* q,
                             float* out, float* pooled_logits, int32_t pool_mode, void* stream) {
  return decode_common(s, c, layer, q, out, pooled_logits, pool_mode, false, stream);
}

SFI_API int sfi_sparse_decode(const sfi_shape* s, const sfi_cache* c, int32_t layer, const float* q,
                              float* out, void* stream) {
  return fast_common(s, c, layer, q, nullptr, nullptr, out, 0, stream);
}

SFI_API int sfi_fast_decode(const sfi_shape* s, const sfi_cache* c, int32_t layer, const float* q,
                            const void* k_new, const void* v_new, float* out, int32_t flags, void* stream) {
  if (!k_new || !v_new) return fail(SFI_ERR_INVALID_ARGUMENT, "fast_decode: k/v null");
  return fast_common(s, c, layer, q, k_new, v_new, out, flags, stream);
}

static int check_selector_params(const sfi_selector_params* prm) {
  // SelectorConfig::validate (config.cpp:68-87)
  const bool ok = prm->alpha > 0.0 && prm->alpha <= 1.0 && prm->gamma >= 0.0 && prm->beta >= 0.0 &&
                  prm->p_curve >= 1.0 && prm->eta >= 0.0 && prm->lambda_clip >= 0.0 &&
                  prm->lambda_clip <= 1.0 && prm->alpha_soft >= 0.0 && prm->alpha_cross >= 0.0 &&
                  prm->temperature > 0.0 && prm->nms_radius >= 0 && prm->epsilon > 0.0 &&
                  std::isfinite(prm->alpha) && std::isfinite(prm->gamma) && std::isfinite(prm->beta) &&
                  std::isfinite(prm->p_curve) && std::isfinite(prm->eta) &&
                  std::isfinite(prm->alpha_soft) && std::isfinite(prm->alpha_cross) &&
                  std::isfinite(prm->temperature) && std::isfinite(prm->epsilon);
  return ok ? SFI_OK : fail(SFI_ERR_CONFIG, "selector: invalid SelectorConfig");
}

static int selector_common(const sfi_shape* s, const sfi_cache* c, int32_t layer, const float* logits,
                           const sfi_selector_params* prm, int phases, const double* z_all, int n_shards,
                           int shard, void* stream, int W = 1) {
  g_launches = 0;
  int rc = validate(s);
  if (rc || (rc = check_cache(s, c)) || (rc = check_layer(s, layer))) return rc;
  if (!prm || ((phases & 1) && !logits)) return fail(SFI_ERR_INVALID_ARGUMENT, "selector: null argument");
  if ((rc = check_selector_params(prm))) return rc;
  if (z_all && (n_shards < 1 || shard < 0 || shard >= n_shards || n_shards * s->n_kv_heads > 16))
    return fail(SFI_ERR_INVALID_ARGUMENT, "selector: bad shard layout (at most 16 heads in total)");
  sfi_impl::Workspace ws = sfi_impl::carve_workspace(*s, c->workspace);
  int n = 0;
  SFI_CUDA(sfi_impl::launch_selector(*s, *c, layer, logits, *prm, ws.sel, (cudaStream_t)stream, &n, phases,
                                     z_all, n_shards, shard, W),
           "sfi_selector");
  g_launches = n;
  return SFI_OK;
}

SFI_API int sfi_selector(const sfi_shape* s, const sfi_cache* c, int32_t layer,
                         const float* pooled_logits, const sfi_selector_params* prm, void* stream) {
  return selector_common(s, c, layer, pooled_logits, prm, 3, nullptr, 1, 0, stream);
}

SFI_API int sfi_selector_window(const sfi_shape* s, const sfi_cache* c, int32_t layer, const float* logits,
                                int32_t W, const sfi_selector_params* prm, void* stream) {
  if (W < 1) return fail(SFI_ERR_OUT_OF_RANGE, "evidence_from_window: window width must be >= 1");
  if (W > 16) return fail(SFI_ERR_UNSUPPORTED, "selector: window width <= 16");
  return selector_common(s, c, layer, logits, prm, 3, nullptr, 1, 0, stream, W);
}

SFI_API int sfi_prefill_capture(const sfi_shape* s, const sfi_cache* c, int32_t layer, const float* q, int32_t W,
                                const int32_t* q_pos, float* logits_out, int32_t pool_mode, void* stream) {
  g_launches = 0;
  int rc = validate(s);
  if (rc || (rc = check_cache(s, c)) || (rc = check_layer(s, layer))) return rc;
  if (!q || !q_pos || !logits_out) return fail(SFI_ERR_INVALID_ARGUMENT, "prefill_capture: null argument");
  if (W < 1 || W > 16) return fail(SFI_ERR_UNSUPPORTED, "prefill_capture: window rows 1..16");
  if (pool_mode != SFI_POOL_MEAN && pool_mode != SFI_POOL_MAX) return fail(SFI_ERR_CONFIG, "prefill_capture: bad pool mode");
  sfi_impl::CaptureParams p;
  p.q = q;
  p.q_pos = q_pos;
  p.k_cache = static_cast<const __nv_bfloat16*>(c->k_cache);
  p.out = logits_out;
  p.prefix_len = c->prefix_len;
  p.n_sink_b = c->n_sink_b;
  p.recent_len = c->recent_len;
  p.layer = layer;
  p.B = s->batch;
  p.H = s->n_kv_heads;
  p.Hq = s->n_q_heads;
  p.Lmax = s->max_positions;
  p.W = W;
  p.pool = pool_mode;
  p.inv_sqrt_d = (float)(1.0 / std::sqrt((double)s->head_dim));
  SFI_CUDA(sfi_impl::launch_capture(p, s->head_dim, (cudaStream_t)stream), "sfi_prefill_capture");
  g_launches = 1;
  return SFI_OK;
}

SFI_API int sfi_selector_fuse(const sfi_shape* s, const sfi_cache* c, int32_t layer,
                              const float* pooled_logits, const sfi_selector_params* prm,
                              const double** z_local, size_t* z_bytes, void* stream) {
  const int rc = selector_common(s, c, layer, pooled_logits, prm, 1, nullptr, 1, 0, stream);
  if (rc) return rc;
  sfi_impl::Workspace ws = sfi_impl::carve_workspace(*s, c->workspace);
  if (z_local) *z_local = ws.sel.a;
  if (z_bytes) *z_bytes = (size_t)s->batch * s->n_kv_heads * s->max_positions * sizeof(double);
  return SFI_OK;
}

SFI_API int sfi_selector_finish(const sfi_shape* s, const sfi_cache* c, int32_t layer,
                                const sfi_selector_params* prm, const double* z_all, int32_t n_shards,
                                int32_t shard, void* stream) {
  if (!z_all) return fail(SFI_ERR_INVALID_ARGUMENT, "selector_finish: z_all is null");
  return selector_common(s, c, layer, nullptr, prm, 2, z_all, n_shards, shard, stream);
}

// ---- sequence sharding ----------------------------------

SFI_API int sfi_seq_lengths(const sfi_shape* s, const sfi_cache* c, int32_t* g_prefix_len,
                            const int32_t* g_n_sink, int32_t* g_recent_len, int32_t advance, int32_t pos_base,
                            int32_t is_last, int32_t* j_off, int32_t* n_glob, void* stream) {
  g_launches = 0;
  int rc = validate(s);
  if (rc || (rc = check_cache(s, c))) return rc;
  if (!g_prefix_len || !g_n_sink || !g_recent_len || !j_off || !n_glob)
    return fail(SFI_ERR_INVALID_ARGUMENT, "seq_lengths: null argument");
  if (pos_base < 0 || advance < 0) return fail(SFI_ERR_INVALID_ARGUMENT, "seq_lengths: negative base/advance");
  SFI_CUDA(sfi_impl::launch_seq_lengths(*s, *c, g_prefix_len, g_n_sink, g_recent_len, advance, pos_base,
                                        is_last ? 1 : 0, j_off, n_glob, (cudaStream_t)stream),
           "sfi_seq_lengths");
  g_launches = 1;
  return SFI_OK;
}

SFI_API int sfi_dense_decode_ex(const sfi_shape* s, const sfi_cache* c, int32_t layer, const float* q, float* out,
                                float* lse, float* pooled_logits, int32_t pool_mode, int32_t flags, void* stream) {
  if (flags & ~(SFI_DENSE_SHARE_SM | SFI_DENSE_TC | SFI_DENSE_MMA))
    return fail(SFI_ERR_INVALID_ARGUMENT, "dense_decode_ex: unknown flags");
  return decode_common(s, c, layer, q, out, pooled_logits, pool_mode, false, stream, lse, flags);
}

SFI_API int sfi_dense_decode_partial(const sfi_shape* s, const sfi_cache* c, int32_t layer, const float* q,
                                     float* out, float* lse, float* pooled_logits, int32_t pool_mode,
                                     void* stream) {
  if (!lse) return fail(SFI_ERR_INVALID_ARGUMENT, "dense_decode_partial: lse is null");
  return decode_common(s, c, layer, q, out, pooled_logits, pool_mode, false, stream, lse);
}

SFI_API int sfi_fast_decode_partial(const sfi_shape* s, const sfi_cache* c, int32_t layer, const float* q,
                                    const void* k_new, const void* v_new, float* out, float* lse, int32_t flags,
                                    void* stream) {
  if (!lse) return fail(SFI_ERR_INVALID_ARGUMENT, "fast_decode_partial: lse is null");
  return fast_common(s, c, layer, q, k_new, v_new, out, flags, stream, lse);
}

SFI_API int sfi_merge_partials(int32_t n_parts, int32_t rows, int32_t head_dim, const float* o_parts,
                               const float* lse_parts, float* out, void* stream) {
  g_launches = 0;
  if (n_parts < 1 || rows < 0 || head_dim < 1 || !o_parts || !lse_parts || !out)
    return fail(SFI_ERR_INVALID_ARGUMENT, "merge_partials: bad argument");
  if (rows == 0) return SFI_OK;
  SFI_CUDA(sfi_impl::launch_merge_partials(n_parts, rows, head_dim, o_parts, lse_parts, out,
                                           (cudaStream_t)stream),
           "sfi_merge_partials");
  g_launches = 1;
  return SFI_OK;
}

SFI_API int sfi_peer_publish(int32_t* flag, void* stream) {
  g_launches = 0;
  if (!flag) return fail(SFI_ERR_INVALID_ARGUMENT, "peer_publish: null flag");
  SFI_CUDA(sfi_impl::launch_peer_publish(flag, (cudaStream_t)stream), "sfi_peer_publish");
  g_launches = 1;
  return SFI_OK;
}

SFI_API int sfi_peer_gather(int32_t n_parts, int64_t bytes, const void* const* src_ptrs,
                            const int32_t* const* flag_ptrs, const int32_t* my_flag, void* dst, void* stream) {
  g_launches = 0;
  if (n_parts < 1 || bytes < 0 || (bytes & 3) || !src_ptrs || !flag_ptrs || !my_flag || !dst)
    return fail(SFI_ERR_INVALID_ARGUMENT, "peer_gather: bad argument (bytes must be a multiple of 4)");
  if (bytes == 0) return SFI_OK;
  SFI_CUDA(sfi_impl::launch_peer_gather(n_parts, bytes / 4, reinterpret_cast<const uint32_t* const*>(src_ptrs),
                                        flag_ptrs, my_flag, static_cast<uint32_t*>(dst), (cudaStream_t)stream),
           "sfi_peer_gather");
  g_launches = 1;
  return SFI_OK;
}

SFI_API int sfi_peer_merge(int32_t n_parts, int32_t rows, int32_t head_dim, const float* const* o_ptrs,
                           const float* const* lse_ptrs, const int32_t* const* flag_ptrs, const int32_t* my_flag,
                           float* out, void* stream) {
  g_launches = 0;
  if (n_parts < 1 || n_parts > sfi_impl::kMaxPeers || rows < 0 || head_dim < 1 || !o_ptrs || !lse_ptrs ||
      !flag_ptrs || !my_flag || !out)
    return fail(SFI_ERR_INVALID_ARGUMENT, "peer_merge: bad argument");
  if (rows == 0) return SFI_OK;
  SFI_CUDA(sfi_impl::launch_peer_merge(n_parts, rows, head_dim, o_ptrs, lse_ptrs, flag_ptrs, my_flag, out,
                                       (cudaStream_t)stream),
           "sfi_peer_merge");
  g_launches = 1;
  return SFI_OK;
}

static int seq_selector_check(const sfi_shape* s, const sfi_cache* c, int32_t layer,
                              const sfi_selector_params* prm) {
  int rc = validate(s);
  if (rc || (rc = check_cache(s, c)) || (rc = check_layer(s, layer))) return rc;
  if (!prm) return fail(SFI_ERR_INVALID_ARGUMENT, "seq_selector: null params");
  if ((rc = check_selector_params(prm))) return rc;
  if (prm->alpha != 1.0)
    return fail(SFI_ERR_UNSUPPORTED, "seq_selector: sequence sharding runs the decode path (W = 1, alpha = 1)");
  if (prm->nms_radius > 16) return fail(SFI_ERR_UNSUPPORTED, "seq_selector: nms_radius <= 16");
  return SFI_OK;
}

SFI_API size_t sfi_seq_edges_doubles(const sfi_shape* s, const sfi_selector_params* prm) {
  if (!s || !prm) return 0;
  return (size_t)s->batch * s->n_kv_heads * (2 * prm->nms_radius + 2);
}

SFI_API int sfi_seq_selector_stats(const sfi_shape* s, const sfi_cache* c, int32_t layer,
                                   const float* pooled_logits, const sfi_selector_params* prm,
                                   const int32_t* j_off, const int32_t* n_glob, int32_t phase, double* row_stats,
                                   const double* stats_all, int32_t n_shards, double* edges, void* stream) {
  g_launches = 0;
  int rc = seq_selector_check(s, c, layer, prm);
  if (rc) return rc;
  if (phase != 1 && phase != 3) return fail(SFI_ERR_INVALID_ARGUMENT, "seq_selector_stats: phase 1 or 3");
  if (!j_off || !n_glob || !row_stats || !pooled_logits ||
      (phase == 3 && (!stats_all || !edges || n_shards < 1)))
    return fail(SFI_ERR_INVALID_ARGUMENT, "seq_selector_stats: null argument");
  sfi_impl::Workspace ws = sfi_impl::carve_workspace(*s, c->workspace);
  SFI_CUDA(sfi_impl::launch_seq_selector_stats(*s, *c, layer, pooled_logits, *prm, ws.sel, j_off, n_glob, phase,
                                               row_stats, stats_all, n_shards, edges, (cudaStream_t)stream),
           "sfi_seq_selector_stats");
  g_launches = 1;
  return SFI_OK;
}

SFI_API int sfi_seq_selector_finish(const sfi_shape* s, const sfi_cache* c, int32_t layer,
                                    const sfi_selector_params* prm, const int32_t* j_off, const int32_t* n_glob,
                                    const double* edges_all, int32_t n_shards, int32_t pos_base,
                                    double* cand_score, int32_t* cand_pos, void* stream) {
  g_launches = 0;
  int rc = seq_selector_check(s, c, layer, prm);
  if (rc) return rc;
  if (!j_off || !n_glob || !edges_all || !cand_score || !cand_pos || n_shards < 1)
    return fail(SFI_ERR_INVALID_ARGUMENT, "seq_selector_finish: bad argument");
  sfi_impl::Workspace ws = sfi_impl::carve_workspace(*s, c->workspace);
  int n = 0;
  SFI_CUDA(sfi_impl::launch_seq_selector_finish(*s, *c, layer, *prm, ws.sel, j_off, n_glob, edges_all, n_shards,
                                                pos_base, cand_score, cand_pos, (cudaStream_t)stream, &n),
           "sfi_seq_selector_finish");
  g_launches = n;
  return SFI_OK;
}

SFI_API size_t sfi_seq_pick_scratch_bytes(const sfi_shape* s, int32_t n_shards) {
  if (!s || n_shards < 1) return 0;
  return sfi_impl::seq_pick_scratch_bytes(*s, n_shards);
}

SFI_API int sfi_seq_selector_pick(const sfi_shape* s, const sfi_cache* c, int32_t layer, int32_t n_shards,
                                  const double* cand_score_all, const int32_t* cand_pos_all, int32_t pos_base,
                                  int32_t pos_end, void* scratch, void* stream) {
  g_launches = 0;
  int rc = validate(s);
  if (rc || (rc = check_cache(s, c)) || (rc = check_layer(s, layer))) return rc;
  if (n_shards < 1 || !cand_score_all || !cand_pos_all || !scratch)
    return fail(SFI_ERR_INVALID_ARGUMENT, "seq_selector_pick: bad argument");
  int n = 0;
  SFI_CUDA(sfi_impl::launch_seq_selector_pick(*s, *c, layer, n_shards, cand_score_all, cand_pos_all, pos_base,
                                              pos_end, scratch, (cudaStream_t)stream, &n),
           "sfi_seq_selector_pick");
  g_launches = n;
  return SFI_OK;
}

SFI_API size_t sfi_selector_explicit_scratch_bytes(int32_t H, int32_t n) {
  return 2 * (size_t)std::max(0, H) * (size_t)std::max(0, n) * sizeof(double);
}

SFI_API int sfi_selector_explicit(int32_t H, int32_t W, int32_t n, int32_t k_budget,
                                  const double* logits, const double* norms, const int32_t* allowed,
                                  const sfi_selector_params* prm, void* scratch, int32_t* sel,
                                  int32_t* n_sel, uint32_t* err, void* stream) {
  g_launches = 0;
  if (H < 1 || H > 16) return fail(SFI_ERR_UNSUPPORTED, "selector: 1..16 heads");
  if (W < 1) return fail(SFI_ERR_OUT_OF_RANGE, "evidence_from_window: window width must be >= 1");
  if (W > 16) return fail(SFI_ERR_UNSUPPORTED, "selector: window width <= 16");
  if (n < 1) return fail(SFI_ERR_EMPTY_SUPPORT, "make_cache_stats: empty allowed set");
  if (k_budget < 0) return fail(SFI_ERR_OUT_OF_RANGE, "select_top_k: negative budget");
  if (!logits || !norms || !allowed || !prm || !scratch || !sel || !n_sel)
    return fail(SFI_ERR_INVALID_ARGUMENT, "selector: null argument");
  double* sa = static_cast<double*>(scratch);
  double* sb = sa + (size_t)H * n;
  int nl = 0;
  SFI_CUDA(sfi_impl::launch_selector_explicit(H, W, n, k_budget, logits, norms, allowed, *prm, sa, sb, sel,
                                              n_sel, err, (cudaStream_t)stream, &nl),
           "sfi_selector_explicit");
  g_launches = nl;
  return SFI_OK;
}

SFI_API int sfi_select_top_k(int32_t rows, int32_t n, int32_t k, const double* scores,
                             const int32_t* allowed, int32_t* sel, int32_t* n_sel, void* stream) {
  g_launches = 0;
  if (k < 0) return fail(SFI_ERR_OUT_OF_RANGE, "select_top_k: negative budget");
  if (rows < 1 || n < 0) return fail(SFI_ERR_INVALID_ARGUMENT, "select_top_k: bad shape");
  if (n > 0 && (!scores || !allowed)) return fail(SFI_ERR_INVALID_ARGUMENT, "select_top_k: null argument");
  int nl = 0;
  SFI_CUDA(sfi_impl::launch_topk_explicit(rows, n, k, scores, allowed, sel, n_sel, (cudaStream_t)stream, &nl),
           "sfi_select_top_k");
  g_launches = nl;
  return SFI_OK;
}

SFI_API int sfi_selector_stage(int32_t stage, int32_t H, int32_t W, int32_t n, const double* a, const double* b,
                               const sfi_selector_params* prm, double* out, double* out2, int32_t* head_err,
                               void* stream) {
  g_launches = 0;
  if (stage < SFI_STAGE_EVIDENCE || stage > SFI_STAGE_CROSS_HEAD)
    return fail(SFI_ERR_INVALID_ARGUMENT, "selector_stage: unknown stage");
  if (H < 0 || n < 0 || (stage == SFI_STAGE_EVIDENCE && W < 1))
    return fail(SFI_ERR_INVALID_ARGUMENT, "selector_stage: bad shape");
  if (H == 0 || n == 0) return SFI_OK;
  const bool needs_b = stage == SFI_STAGE_PRIOR || stage == SFI_STAGE_FUSE;
  const bool needs_err = stage <= SFI_STAGE_NORMALIZE;
  if (!a || !out || !prm || (needs_b && !b) || (needs_err && !head_err))
    return fail(SFI_ERR_INVALID_ARGUMENT, "selector_stage: null argument");
  SFI_CUDA(sfi_impl::launch_selector_stage(stage, H, W, n, a, b, *prm, out, out2, head_err, (cudaStream_t)stream),
           "sfi_selector_stage");
  g_launches = 1;
  return SFI_OK;
}

SFI_API int sfi_selector_stages(const sfi_shape* s, const sfi_cache* c, int32_t b, double* z_base,
                                double* z_adj, int32_t n_j, void* stream) {
  int rc = validate(s);
  if (rc || (rc = check_cache(s, c))) return rc;
  if (b < 0 || b >= s->batch || n_j < 0 || n_j > s->max_positions)
    return fail(SFI_ERR_OUT_OF_RANGE, "selector_stages: bad request index or length");
  sfi_impl::Workspace ws = sfi_impl::carve_workspace(*s, c->workspace);
  cudaStream_t st = (cudaStream_t)stream;
  for (int h = 0; h < s->n_kv_heads; ++h) {
    const size_t off = ((size_t)b * s->n_kv_heads + h) * s->max_positions;
    if (z_base)
      SFI_CUDA(cudaMemcpyAsync(z_base + (size_t)h * n_j, ws.sel.a + off, n_j * sizeof(double),
                               cudaMemcpyDeviceToHost, st), "selector_stages");
    if (z_adj)
      SFI_CUDA(cudaMemcpyAsync(z_adj + (size_t)h * n_j, ws.sel.b + off, n_j * sizeof(double),
                               cudaMemcpyDeviceToHost, st), "selector_stages");
  }
  SFI_CUDA(cudaStreamSynchronize(st), "selector_stages");
  return SFI_OK;
}

SFI_API int sfi_compact_build(const sfi_shape* s, const sfi_cache* c, int32_t layer,
                              int32_t rebuild_ring, void* stream) {
  g_launches = 0;
  int rc = validate(s);
  if (rc || (rc = check_cache(s, c)) || (rc = check_layer(s, layer))) return rc;
  SFI_CUDA(sfi_impl::launch_compact_build(*s, *c, layer, rebuild_ring, (cudaStream_t)stream),
           "sfi_compact_build");
  g_launches = 1;
  return SFI_OK;
}

SFI_API int sfi_set_selection(const sfi_shape* s, const sfi_cache* c, int32_t layer,
                              const int32_t* sel_host, const int32_t* counts_host, void* stream) {
  g_launches = 0;
  int rc = validate(s);
  if (rc || (rc = check_cache(s, c)) || (rc = check_layer(s, layer))) return rc;
  if (!counts_host || (!sel_host && s->k_budget > 0))
    return fail(SFI_ERR_INVALID_ARGUMENT, "set_selection: null argument");
  const size_t slices = (size_t)s->batch * s->n_kv_heads;
  for (size_t i = 0; i < slices; ++i)
    if (counts_host[i] < 0 || counts_host[i] > s->k_budget)
      return fail(SFI_ERR_OUT_OF_RANGE, "set_selection: selected set exceeds k_budget");
  cudaStream_t st = (cudaStream_t)stream;
  if (s->k_budget > 0)
    SFI_CUDA(cudaMemcpyAsync(c->sel + (size_t)layer * slices * s->k_budget, sel_host,
                             slices * s->k_budget * sizeof(int32_t), cudaMemcpyHostToDevice, st),
             "set_selection");
  SFI_CUDA(cudaMemcpyAsync(c->n_sel + (size_t)layer * slices, counts_host, slices * sizeof(int32_t),
                           cudaMemcpyHostToDevice, st),
           "set_selection");
  SFI_CUDA(sfi_impl::launch_compact_build(*s, *c, layer, 0, st), "set_selection");
  SFI_CUDA(cudaStreamSynchronize(st), "set_selection");
  g_launches = 1;
  return SFI_OK;
}

SFI_API int sfi_read_errors(const sfi_cache* c, uint32_t* flags_out, void* stream) {
  if (!c || !c->error_flags) return fail(SFI_ERR_INVALID_ARGUMENT, "read_errors: null cache");
  cudaStream_t st = (cudaStream_t)stream;
  uint32_t f = 0;
  SFI_CUDA(cudaMemcpyAsync(&f, c->error_flags, sizeof(f), cudaMemcpyDeviceToHost, st), "read_errors");
  SFI_CUDA(cudaStreamSynchronize(st), "read_errors");
  if (f) SFI_CUDA(cudaMemsetAsync(c->error_flags, 0, sizeof(uint32_t), st), "read_errors");
  SFI_CUDA(cudaStreamSynchronize(st), "read_errors");
  if (flags_out) *flags_out = f;
  if (!f) return SFI_OK;
  for (int code = 1; code < 32; ++code)
    if (f & (1u << code)) {
      static const char* names[] = {"ok", "config", "empty_support", "support_mismatch",
                                    "non_finite_input", "overlap_violation", "stale_compact",
                                    "out_of_range", "bad_weight_file", "context_overflow", "io"};
      return fail(code, std::string("device contract violation: ") + (code <= 10 ? names[code] : "?"));
    }
  return SFI_OK;
}

SFI_API int sfi_fill_synthetic(const sfi_shape* s, const sfi_cache* c, uint64_t seed, int32_t len,
                               void* stream) {
  g_launches = 0;
  int rc = validate(s);
  if (rc || (rc = check_cache(s, c))) return rc;
  if (len < 0 || len > s->max_positions) return fail(SFI_ERR_OUT_OF_RANGE, "fill_synthetic: bad length");
  SFI_CUDA(sfi_impl::launch_fill_synthetic(*s, *c, seed, len, (cudaStream_t)stream), "sfi_fill_synthetic");
  g_launches = 2;
  return SFI_OK;
}

}  // extern "C"

// ---- multi-GPU entry points over an NCCL communicator ----
// The exchange of each sharded step, done in-call on `stream`: the caller
// passes an ncclComm_t (from ncclCommInitRank, or torch's ProcessGroupNCCL
// communicator). NCCL is resolved at run time from the process — the library
// that created the communicator (RTLD_DEFAULT), else libnccl.so.2 — so
// libsfi_b200.so carries no link-time NCCL dependency and never mixes two NCCL
// builds in one process.
namespace {

using NcclAllGather = int (*)(const void*, void*, size_t, int, void*, cudaStream_t);
using NcclErrStr = const char* (*)(int);
constexpr int kNcclInt32 = 2, kNcclFloat32 = 7, kNcclFloat64 = 8;  // ncclDataType_t (nccl.h)

struct NcclApi {
  NcclAllGather all_gather = nullptr;
  NcclErrStr err_str = nullptr;
};

const NcclApi& nccl_api() {
  static const NcclApi api = [] {
    NcclApi a;
    void* f = dlsym(RTLD_DEFAULT, "ncclAllGather");
    void* e = dlsym(RTLD_DEFAULT, "ncclGetErrorString");
    if (!f) {
      void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
      if (h) {
        f = dlsym(h, "ncclAllGather");
        e = dlsym(h, "ncclGetErrorString");
      }
    }
    a.all_gather = reinterpret_cast<NcclAllGather>(f);
    a.err_str = reinterpret_cast<NcclErrStr>(e);
    return a;
  }();
  return api;
}

int nccl_gather(const void* send, void* recv, size_t count, int dtype, void* comm, void* stream, const char* what) {
  const NcclApi& api = nccl_api();
  if (!api.all_gather) return fail(SFI_ERR_UNSUPPORTED, std::string(what) + ": NCCL is not available in this process");
  const int r = api.all_gather(send, recv, count, dtype, comm, (cudaStream_t)stream);
  if (r != 0)
    return fail(SFI_ERR_CUDA, std::string(what) + ": ncclAllGather failed: " + (api.err_str ? api.err_str(r) : "?"));
  return SFI_OK;
}

size_t al256(size_t x) { return (x + 255) & ~size_t(255); }

}  // namespace

SFI_API int sfi_selector_sharded_nccl(const sfi_shape* s, const sfi_cache* c, int32_t layer, const float* logits,
                                      const sfi_selector_params* prm, void* comm, int32_t n_shards, int32_t shard,
                                      double* z_all, void* stream) {
  if (!comm || !z_all) return fail(SFI_ERR_INVALID_ARGUMENT, "selector_sharded_nccl: null communicator or z_all");
  if (n_shards < 1 || shard < 0 || shard >= n_shards)
    return fail(SFI_ERR_INVALID_ARGUMENT, "selector_sharded_nccl: bad shard index");
  const double* z = nullptr;
  size_t bytes = 0;
  int rc = sfi_selector_fuse(s, c, layer, logits, prm, &z, &bytes, stream);
  if (rc) return rc;
  const int nl = g_launches;
  if ((rc = nccl_gather(z, z_all, bytes / sizeof(double), kNcclFloat64, comm, stream, "selector_sharded_nccl")))
    return rc;
  rc = sfi_selector_finish(s, c, layer, prm, z_all, n_shards, shard, stream);
  g_launches += nl;
  return rc;
}

SFI_API int sfi_merge_partials_nccl(int32_t n_parts, int32_t rows, int32_t head_dim, const float* o_part,
                                    const float* lse_part, float* o_all, float* lse_all, float* out, void* comm,
                                    void* stream) {
  if (!comm || !o_part || !lse_part || !o_all || !lse_all || !out)
    return fail(SFI_ERR_INVALID_ARGUMENT, "merge_partials_nccl: null argument");
  int rc = nccl_gather(o_part, o_all, (size_t)rows * head_dim, kNcclFloat32, comm, stream, "merge_partials_nccl");
  if (rc || (rc = nccl_gather(lse_part, lse_all, (size_t)rows, kNcclFloat32, comm, stream, "merge_partials_nccl")))
    return rc;
  return sfi_merge_partials(n_parts, rows, head_dim, o_all, lse_all, out, stream);
}

namespace {
struct SeqNcclScratch {
  double *row_stats, *stats_all, *edges, *edges_all, *cand_score, *cand_score_all;
  int32_t *cand_pos, *cand_pos_all;
  void* pick;
  size_t bytes;
};
SeqNcclScratch seq_nccl_layout(const sfi_shape* s, const sfi_selector_params* prm, int32_t P, void* base) {
  const size_t rows = (size_t)s->batch * s->n_kv_heads, K = (size_t)std::max(s->k_budget, 1);
  const size_t ne = (size_t)sfi_seq_edges_doubles(s, prm);
  uint8_t* p = static_cast<uint8_t*>(base);
  SeqNcclScratch x{};
  size_t off = 0;
  auto take = [&](size_t bytes) {
    void* q = p ? p + off : nullptr;
    off += al256(bytes);
    return q;
  };
  x.row_stats = static_cast<double*>(take(rows * 6 * 8));
  x.stats_all = static_cast<double*>(take(P * rows * 6 * 8));
  x.edges = static_cast<double*>(take(ne * 8));
  x.edges_all = static_cast<double*>(take(P * ne * 8));
  x.cand_score = static_cast<double*>(take(rows * K * 8));
  x.cand_score_all = static_cast<double*>(take(P * rows * K * 8));
  x.cand_pos = static_cast<int32_t*>(take(rows * K * 4));
  x.cand_pos_all = static_cast<int32_t*>(take(P * rows * K * 4));
  x.pick = take(sfi_seq_pick_scratch_bytes(s, P));
  x.bytes = off;
  return x;
}
}  // namespace

SFI_API size_t sfi_seq_selector_nccl_scratch_bytes(const sfi_shape* s, const sfi_selector_params* prm,
                                                   int32_t n_shards) {
  if (!s || !prm || n_shards < 1) return 0;
  return seq_nccl_layout(s, prm, n_shards, nullptr).bytes;
}

SFI_API int sfi_seq_selector_nccl(const sfi_shape* s, const sfi_cache* c, int32_t layer, const float* logits,
                                  const sfi_selector_params* prm, const int32_t* j_off, const int32_t* n_glob,
                                  int32_t pos_base, int32_t pos_end, void* comm, int32_t n_shards, void* scratch,
                                  size_t scratch_bytes, void* stream) {
  if (!comm || !scratch || !prm) return fail(SFI_ERR_INVALID_ARGUMENT, "seq_selector_nccl: null argument");
  const SeqNcclScratch x = seq_nccl_layout(s, prm, n_shards, scratch);
  if (scratch_bytes < x.bytes) return fail(SFI_ERR_INVALID_ARGUMENT, "seq_selector_nccl: scratch too small");
  const size_t rows = (size_t)s->batch * s->n_kv_heads, K = (size_t)std::max(s->k_budget, 1);
  const size_t ne = (size_t)sfi_seq_edges_doubles(s, prm);
  int launches = 0, rc;
  // row statistics -> global max / sums; soft-NMS edges; top-k candidates -> global pick
  if ((rc = sfi_seq_selector_stats(s, c, layer, logits, prm, j_off, n_glob, 1, x.row_stats, x.stats_all, n_shards,
                                   x.edges, stream)))
    return rc;
  launches += g_launches;
  if ((rc = nccl_gather(x.row_stats, x.stats_all, rows * 6, kNcclFloat64, comm, stream, "seq_selector_nccl"))) return rc;
  if ((rc = sfi_seq_selector_stats(s, c, layer, logits, prm, j_off, n_glob, 3, x.row_stats, x.stats_all, n_shards,
                                   x.edges, stream)))
    return rc;
  launches += g_launches;
  if ((rc = nccl_gather(x.edges, x.edges_all, ne, kNcclFloat64, comm, stream, "seq_selector_nccl"))) return rc;
  if ((rc = sfi_seq_selector_finish(s, c, layer, prm, j_off, n_glob, x.edges_all, n_shards, pos_base, x.cand_score,
                                    x.cand_pos, stream)))
    return rc;
  launches += g_launches;
  if ((rc = nccl_gather(x.cand_score, x.cand_score_all, rows * K, kNcclFloat64, comm, stream, "seq_selector_nccl")) ||
      (rc = nccl_gather(x.cand_pos, x.cand_pos_all, rows * K, kNcclInt32, comm, stream, "seq_selector_nccl")))
    return rc;
  rc = sfi_seq_selector_pick(s, c, layer, n_shards, x.cand_score_all, x.cand_pos_all, pos_base, pos_end, x.pick,
                             stream);
  g_launches += launches;
  return rc;
}

SFI_API int sfi_launch_floor(int32_t n_launches, int32_t grid, void* stream) {
  g_launches = 0;
  if (n_launches < 0 || grid < 1) return fail(SFI_ERR_INVALID_ARGUMENT, "launch_floor: bad arguments");
  SFI_CUDA(sfi_impl::launch_floor(n_launches, grid, (cudaStream_t)stream), "sfi_launch_floor");
  g_launches = n_launches;
  return SFI_OK;
}

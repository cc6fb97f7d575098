// host.cpp — C++ host API (include/sfi_b200.hpp): the reference's operator
// interface re-expressed over the C ABI. Host code here only validates
// arguments (with the reference's error codes, in the reference's order),
// stages host vectors to/from HBM and launches the device path; all hot-path
// arithmetic runs in the sm_100a kernels.
#include "sfi_b200.hpp"

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <iterator>
#include <numeric>

namespace sfi_b200 {

namespace {

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) fail(ErrorCode::kCuda, std::string(what) + ": " + cudaGetErrorString(e));
}

cudaStream_t st(void* s) { return static_cast<cudaStream_t>(s); }

// Grow-only device scratch owned by the calling thread.
struct Scratch {
  void* p = nullptr;
  size_t n = 0;
  void* get(size_t bytes) {
    if (bytes > n) {
      if (p) cudaFree(p);
      p = nullptr;
      n = 0;
      cuda_check(cudaMalloc(&p, bytes), "scratch alloc");
      n = bytes;
    }
    return p;
  }
  ~Scratch() {
    if (p) cudaFree(p);
  }
};
thread_local Scratch t_scratch;

size_t al(size_t x) { return (x + 255) & ~size_t(255); }

uint16_t to_bf16(float x) {
  const __nv_bfloat16 b = __float2bfloat16_rn(x);
  uint16_t u;
  std::memcpy(&u, &b, 2);
  return u;
}
float from_bf16(uint16_t u) {
  uint32_t w = static_cast<uint32_t>(u) << 16;
  float f;
  std::memcpy(&f, &w, 4);
  return f;
}

void require(bool ok, const char* what) {
  if (!ok) fail(ErrorCode::kConfig, what);
}

}  // namespace

// ---------------------------------------------------------------------------
// errors

void fail(ErrorCode code, const std::string& message) { throw Error(code, message); }

void check(int status) {
  if (status == SFI_OK) return;
  const std::string msg = sfi_last_error();
  if (status >= 1 && status <= 10) fail(static_cast<ErrorCode>(status - 1), msg);
  if (status == SFI_ERR_UNSUPPORTED) fail(ErrorCode::kUnsupported, msg);
  if (status == SFI_ERR_INVALID_ARGUMENT) fail(ErrorCode::kOutOfRange, msg);
  fail(ErrorCode::kCuda, msg);
}

const char* error_code_name(ErrorCode code) {
  switch (code) {
    case ErrorCode::kConfig: return "config";
    case ErrorCode::kEmptySupport: return "empty_support";
    case ErrorCode::kSupportMismatch: return "support_mismatch";
    case ErrorCode::kNonFiniteInput: return "non_finite_input";
    case ErrorCode::kOverlapViolation: return "overlap_violation";
    case ErrorCode::kStaleCompact: return "stale_compact";
    case ErrorCode::kOutOfRange: return "out_of_range";
    case ErrorCode::kBadWeightFile: return "bad_weight_file";
    case ErrorCode::kContextOverflow: return "context_overflow";
    case ErrorCode::kIo: return "io";
    case ErrorCode::kCuda: return "cuda";
    case ErrorCode::kUnsupported: return "unsupported";
  }
  return "unknown";
}

// ---------------------------------------------------------------------------
// config (config.cpp:68-101)

void SelectorConfig::validate() const {
  require(alpha > 0.0 && alpha <= 1.0, "alpha must be in (0, 1]");
  require(gamma >= 0.0, "gamma must be >= 0");
  require(beta >= 0.0, "beta must be >= 0");
  require(p_curve >= 1.0, "p_curve must be >= 1");
  require(eta >= 0.0, "eta must be >= 0");
  require(lambda_clip >= 0.0 && lambda_clip <= 1.0, "lambda_clip must be in [0, 1]");
  require(alpha_soft >= 0.0, "alpha_soft must be >= 0");
  require(alpha_cross >= 0.0, "alpha_cross must be >= 0");
  require(temperature > 0.0, "temperature must be > 0");
  require(nms_radius >= 0, "nms_radius must be >= 0");
  require(epsilon > 0.0, "epsilon must be > 0");
  require(k_budget >= 0, "k_budget must be >= 0");
  for (double v : {alpha, gamma, beta, p_curve, eta, lambda_clip, alpha_soft, alpha_cross,
                   temperature, epsilon})
    require(std::isfinite(v), "selector values must be finite");
}

sfi_selector_params SelectorConfig::to_params() const {
  sfi_selector_params p;
  p.alpha = alpha;
  p.gamma = gamma;
  p.beta = beta;
  p.p_curve = p_curve;
  p.eta = eta;
  p.lambda_clip = lambda_clip;
  p.alpha_soft = alpha_soft;
  p.alpha_cross = alpha_cross;
  p.temperature = temperature;
  p.epsilon = epsilon;
  p.nms_radius = nms_radius;
  p.pool = pool == PoolMode::kMax ? SFI_POOL_MAX : SFI_POOL_MEAN;
  return p;
}

void TriggerConfig::validate() const {
  require(t_max >= 1, "t_max must be >= 1");
  require(window_decode >= 1, "window_decode must be >= 1");
  require(window_prefill >= 1, "window_prefill must be >= 1");
}

bool TriggerConfig::is_trigger(TokenId id) const {
  return std::find(trigger_tokens.begin(), trigger_tokens.end(), id) != trigger_tokens.end();
}

void CacheLimits::validate() const {
  require(n_sink >= 0, "n_sink must be >= 0");
  require(n_recent >= 1, "n_recent must be >= 1");
  require(k_budget >= 0, "k_budget must be >= 0");
}

void Config::validate() const {
  selector.validate();
  trigger.validate();
  limits.validate();
}

Config default_config() { return Config{}; }

void ModelSpec::validate() const {
  auto bad = [](const std::string& what) { fail(ErrorCode::kConfig, "model spec: " + what); };
  if (n_layers < 1) bad("n_layers must be >= 1");
  if (n_query_heads < 1 || n_kv_heads < 1) bad("head counts must be >= 1");
  if (n_query_heads % n_kv_heads != 0) bad("n_query_heads must be a multiple of n_kv_heads");
  if (head_dim < 2 || head_dim % 2 != 0) bad("head_dim must be even and >= 2");
  if (vocab_size < 2) bad("vocab_size must be >= 2");
  if (max_positions < 1) bad("max_positions must be >= 1");
  if (!(rope_base > 0.0)) bad("rope_base must be > 0");
}

// ---------------------------------------------------------------------------
// selector

CacheStats make_cache_stats(std::vector<std::vector<double>> key_norms,
                            const std::vector<Pos>& allowed, double epsilon) {
  if (allowed.empty()) fail(ErrorCode::kEmptySupport, "make_cache_stats: empty allowed set");
  for (const auto& per_head : key_norms)
    if (per_head.size() != allowed.size())
      fail(ErrorCode::kSupportMismatch, "make_cache_stats: key_norms misaligned with J");
  CacheStats stats;
  stats.key_norms = std::move(key_norms);
  stats.j_min = allowed.front();
  stats.j_max = allowed.back();
  stats.normalized_pos.resize(allowed.size());
  const double denom = static_cast<double>(stats.j_max - stats.j_min) + epsilon;
  for (std::size_t i = 0; i < allowed.size(); ++i)
    stats.normalized_pos[i] = static_cast<double>(allowed[i] - stats.j_min) / denom;
  return stats;
}

std::vector<Pos> select_top_k(const std::vector<double>& scores, const std::vector<Pos>& allowed,
                              int k) {
  if (scores.size() != allowed.size())
    fail(ErrorCode::kSupportMismatch, "select_top_k: score/support mismatch");
  if (k < 0) fail(ErrorCode::kOutOfRange, "select_top_k: negative budget");
  const int n = static_cast<int>(scores.size());
  const size_t kk = static_cast<size_t>(std::max(1, std::min(k, std::max(n, 1))));
  const size_t nn = static_cast<size_t>(std::max(n, 1));
  uint8_t* base = static_cast<uint8_t*>(
      t_scratch.get(al(nn * 8) + al(nn * 4) + al(kk * 4) + al(4)));
  double* d_scores = reinterpret_cast<double*>(base);
  int32_t* d_allowed = reinterpret_cast<int32_t*>(base + al(nn * 8));
  int32_t* d_sel = reinterpret_cast<int32_t*>(base + al(nn * 8) + al(nn * 4));
  int32_t* d_cnt = reinterpret_cast<int32_t*>(base + al(nn * 8) + al(nn * 4) + al(kk * 4));
  if (n > 0) {
    cuda_check(cudaMemcpy(d_scores, scores.data(), n * 8, cudaMemcpyHostToDevice), "select_top_k");
    cuda_check(cudaMemcpy(d_allowed, allowed.data(), n * 4, cudaMemcpyHostToDevice), "select_top_k");
  }
  check(sfi_select_top_k(1, n, k, d_scores, d_allowed, d_sel, d_cnt, nullptr));
  int32_t cnt = 0;
  cuda_check(cudaMemcpy(&cnt, d_cnt, 4, cudaMemcpyDeviceToHost), "select_top_k");
  std::vector<Pos> out(static_cast<size_t>(cnt));
  if (cnt) cuda_check(cudaMemcpy(out.data(), d_sel, cnt * 4, cudaMemcpyDeviceToHost), "select_top_k");
  return out;
}

std::vector<std::vector<Pos>> run_selector(const LogitWindow& w, const CacheStats& stats,
                                           const SelectorConfig& cfg, SelectorStages* stages) {
  // argument checks in the reference's order (selector.cpp:258-264, 99-108, 133-143)
  if (w.heads() != static_cast<int>(stats.key_norms.size()))
    fail(ErrorCode::kSupportMismatch, "run_selector: window/stats head count mismatch");
  if (w.allowed.empty()) fail(ErrorCode::kEmptySupport, "evidence_from_window: empty support");
  if (w.width < 1) fail(ErrorCode::kOutOfRange, "evidence_from_window: window width must be >= 1");
  const int H = w.heads();
  const int W = w.width;
  const int n = static_cast<int>(w.allowed.size());
  for (int h = 0; h < H; ++h)
    if (w.values[h].size() != static_cast<size_t>(W) * n)
      fail(ErrorCode::kSupportMismatch, "evidence_from_window: bad window shape");
  if (stats.normalized_pos.size() != w.allowed.size())
    fail(ErrorCode::kSupportMismatch, "prior_from_stats: stats misaligned with J");
  for (int h = 0; h < H; ++h)
    if (stats.key_norms[h].size() != static_cast<size_t>(n))
      fail(ErrorCode::kSupportMismatch, "prior_from_stats: key_norms misaligned with J");
  if (H == 0) return {};
  const int K = cfg.k_budget;
  if (K < 0) fail(ErrorCode::kOutOfRange, "select_top_k: negative budget");
  const size_t hn = static_cast<size_t>(H) * n;
  const size_t kk = static_cast<size_t>(std::max(K, 1));
  const size_t b_logits = al(hn * W * 8), b_norms = al(hn * 8), b_allowed = al(n * 4);
  const size_t b_scr = al(sfi_selector_explicit_scratch_bytes(H, n));
  const size_t b_sel = al(H * kk * 4), b_cnt = al(H * 4), b_err = al(4);
  uint8_t* base = static_cast<uint8_t*>(
      t_scratch.get(b_logits + b_norms + b_allowed + b_scr + b_sel + b_cnt + b_err));
  double* d_logits = reinterpret_cast<double*>(base);
  double* d_norms = reinterpret_cast<double*>(base + b_logits);
  int32_t* d_allowed = reinterpret_cast<int32_t*>(base + b_logits + b_norms);
  void* d_scr = base + b_logits + b_norms + b_allowed;
  int32_t* d_sel = reinterpret_cast<int32_t*>(base + b_logits + b_norms + b_allowed + b_scr);
  int32_t* d_cnt = reinterpret_cast<int32_t*>(base + b_logits + b_norms + b_allowed + b_scr + b_sel);
  uint32_t* d_err =
      reinterpret_cast<uint32_t*>(base + b_logits + b_norms + b_allowed + b_scr + b_sel + b_cnt);
  std::vector<double> flat(hn * W);
  std::vector<double> nflat(hn);
  for (int h = 0; h < H; ++h) {
    std::copy(w.values[h].begin(), w.values[h].end(), flat.begin() + static_cast<size_t>(h) * W * n);
    std::copy(stats.key_norms[h].begin(), stats.key_norms[h].end(), nflat.begin() + static_cast<size_t>(h) * n);
  }
  cuda_check(cudaMemcpy(d_logits, flat.data(), flat.size() * 8, cudaMemcpyHostToDevice), "run_selector");
  cuda_check(cudaMemcpy(d_norms, nflat.data(), nflat.size() * 8, cudaMemcpyHostToDevice), "run_selector");
  cuda_check(cudaMemcpy(d_allowed, w.allowed.data(), n * 4, cudaMemcpyHostToDevice), "run_selector");
  cuda_check(cudaMemset(d_err, 0, 4), "run_selector");
  const sfi_selector_params prm = cfg.to_params();
  check(sfi_selector_explicit(H, W, n, K, d_logits, d_norms, d_allowed, &prm, d_scr, d_sel, d_cnt,
                              d_err, nullptr));
  uint32_t err = 0;
  cuda_check(cudaMemcpy(&err, d_err, 4, cudaMemcpyDeviceToHost), "run_selector");
  if (err & (1u << SFI_ERR_NON_FINITE_INPUT))
    fail(ErrorCode::kNonFiniteInput, "run_selector: non-finite logit or bad key norm");
  if (err & (1u << SFI_ERR_EMPTY_SUPPORT))
    fail(ErrorCode::kEmptySupport, "run_selector: fully masked row or all-zero weights");
  std::vector<int32_t> cnt(H);
  std::vector<int32_t> sel(static_cast<size_t>(H) * kk);
  cuda_check(cudaMemcpy(cnt.data(), d_cnt, H * 4, cudaMemcpyDeviceToHost), "run_selector");
  if (K > 0) cuda_check(cudaMemcpy(sel.data(), d_sel, sel.size() * 4, cudaMemcpyDeviceToHost), "run_selector");
  std::vector<std::vector<Pos>> out(static_cast<size_t>(H));
  for (int h = 0; h < H; ++h)
    out[h].assign(sel.begin() + static_cast<size_t>(h) * kk, sel.begin() + static_cast<size_t>(h) * kk + cnt[h]);
  if (stages) {
    std::vector<double> a(hn), b(hn);
    const double* sa = static_cast<const double*>(d_scr);
    cuda_check(cudaMemcpy(a.data(), sa, hn * 8, cudaMemcpyDeviceToHost), "run_selector");
    cuda_check(cudaMemcpy(b.data(), sa + hn, hn * 8, cudaMemcpyDeviceToHost), "run_selector");
    stages->base.assign(H, {});
    stages->after_cross.assign(H, {});
    for (int h = 0; h < H; ++h) {
      stages->base[h].assign(a.begin() + static_cast<size_t>(h) * n, a.begin() + static_cast<size_t>(h + 1) * n);
      stages->after_cross[h].assign(b.begin() + static_cast<size_t>(h) * n, b.begin() + static_cast<size_t>(h + 1) * n);
    }
  }
  return out;
}

// ---------------------------------------------------------------------------
// device cache

DeviceCache::DeviceCache(const sfi_shape& shape) : shape_(shape) {
  check(sfi_buffer_sizes(&shape_, &sizes_));
  auto alloc = [&](size_t bytes) {
    void* p = nullptr;
    cuda_check(cudaMalloc(&p, std::max<size_t>(bytes, 256)), "DeviceCache alloc");
    cuda_check(cudaMemset(p, 0, std::max<size_t>(bytes, 256)), "DeviceCache memset");
    allocs_.push_back(p);
    return p;
  };
  cache_.k_cache = alloc(sizes_.kv_cache);
  cache_.v_cache = alloc(sizes_.kv_cache);
  cache_.key_norms = static_cast<double*>(alloc(sizes_.key_norms));
  cache_.ck = alloc(sizes_.compact);
  cache_.cv = alloc(sizes_.compact);
  cache_.sel = static_cast<int32_t*>(alloc(sizes_.sel));
  cache_.n_sel = static_cast<int32_t*>(alloc(sizes_.n_sel));
  cache_.prefix_len = static_cast<int32_t*>(alloc(sizes_.per_batch));
  cache_.n_sink_b = static_cast<int32_t*>(alloc(sizes_.per_batch));
  cache_.recent_len = static_cast<int32_t*>(alloc(sizes_.per_batch));
  cache_.error_flags = static_cast<uint32_t*>(alloc(4));
  cache_.workspace = alloc(sizes_.workspace);
  cache_.workspace_bytes = sizes_.workspace;
  logits_ = static_cast<float*>(alloc(sizes_.pooled_logits));
}

DeviceCache::~DeviceCache() {
  for (void* p : allocs_) cudaFree(p);
}

// ---------------------------------------------------------------------------
// KvStore

KvStore::KvStore(const ModelSpec& spec, const CacheLimits& limits, void* stream)
    : spec_(spec), limits_(limits), stream_(stream), layers_(spec.n_layers) {
  spec.validate();
  limits.validate();
  sfi_shape s{};
  s.n_layers = spec.n_layers;
  s.batch = 1;
  s.n_kv_heads = spec.n_kv_heads;
  s.n_q_heads = spec.n_query_heads;
  s.head_dim = spec.head_dim;
  s.max_positions = spec.max_positions;
  s.n_sink = limits.n_sink;
  s.k_budget = limits.k_budget;
  s.n_recent = limits.n_recent;
  check(sfi_shape_validate(&s));
  dev_ = std::make_unique<DeviceCache>(s);
}

void KvStore::set_window(int n_sink_b, int recent_len, Pos len) const {
  if (len < 0) len = len_;
  if (n_sink_b == cur_nsb_ && recent_len == cur_rl_ && len == cur_len_) return;
  const int32_t L = len, nsb = n_sink_b, rl = recent_len;
  check(sfi_set_lengths(&dev_->shape(), &dev_->cache(), &L, &nsb, &rl, stream_));
  cur_nsb_ = n_sink_b;
  cur_rl_ = recent_len;
  cur_len_ = len;
}

std::vector<double> KvStore::key_norms(int layer, int head, Pos first, int count) const {
  std::vector<double> out(static_cast<size_t>(std::max(count, 0)));
  if (count <= 0) return out;
  const Pos visible = len_ + (pending_layers_ > layer ? 1 : 0);
  if (first < 1 || first + count - 1 > visible)
    fail(ErrorCode::kOutOfRange, "KvStore: key norm range not written");
  const size_t off = (static_cast<size_t>(layer) * spec_.n_kv_heads + head) * spec_.max_positions + (first - 1);
  cuda_check(cudaStreamSynchronize(st(stream_)), "key_norms");
  cuda_check(cudaMemcpy(out.data(), dev_->cache().key_norms + off, out.size() * 8, cudaMemcpyDeviceToHost),
             "key_norms");
  return out;
}

void KvStore::begin_token() {
  if (pending_layers_ != -1) fail(ErrorCode::kOutOfRange, "KvStore: token already open");
  if (len_ >= spec_.max_positions) fail(ErrorCode::kContextOverflow, "KvStore: max_positions exceeded");
  pending_layers_ = 0;
}

void KvStore::append_layer(int layer, const float* k, const float* v) {
  if (pending_layers_ != layer) fail(ErrorCode::kOutOfRange, "KvStore: layers must be appended in order");
  const int hd = spec_.n_kv_heads * spec_.head_dim;
  std::vector<uint16_t> hk(hd), hv(hd);
  for (int i = 0; i < hd; ++i) {
    hk[i] = to_bf16(k[i]);
    hv[i] = to_bf16(v[i]);
  }
  set_window(std::max(cur_nsb_, 0), 0);
  uint16_t* d = static_cast<uint16_t*>(t_scratch.get(al(hd * 2) * 2));
  cuda_check(cudaMemcpyAsync(d, hk.data(), hd * 2, cudaMemcpyHostToDevice, st(stream_)), "append_layer");
  cuda_check(cudaMemcpyAsync(d + al(hd * 2) / 2, hv.data(), hd * 2, cudaMemcpyHostToDevice, st(stream_)),
             "append_layer");
  check(sfi_append_block(&dev_->shape(), &dev_->cache(), layer, 1, d, d + al(hd * 2) / 2, stream_));
  cuda_check(cudaStreamSynchronize(st(stream_)), "append_layer");
  ++pending_layers_;
}

void KvStore::end_token() {
  if (pending_layers_ != spec_.n_layers)
    fail(ErrorCode::kOutOfRange, "KvStore: token closed before all layers were appended");
  pending_layers_ = -1;
  ++len_;
}

void KvStore::append_tokens(int count, const float* k, const float* v) {
  if (pending_layers_ != -1) fail(ErrorCode::kOutOfRange, "KvStore: token already open");
  if (count < 0) fail(ErrorCode::kOutOfRange, "KvStore: negative token count");
  if (len_ + count > spec_.max_positions) fail(ErrorCode::kContextOverflow, "KvStore: max_positions exceeded");
  if (count == 0) return;
  const int H = spec_.n_kv_heads, d = spec_.head_dim;
  const size_t per = static_cast<size_t>(count) * H * d;
  std::vector<uint16_t> hk(per), hv(per);
  set_window(std::max(cur_nsb_, 0), 0);
  uint16_t* dk = static_cast<uint16_t*>(t_scratch.get(al(per * 2) * 2));
  uint16_t* dv = dk + al(per * 2) / 2;
  for (int l = 0; l < spec_.n_layers; ++l) {
    // [count][H][d] -> [H][count][d]
    const float* kl = k + static_cast<size_t>(l) * per;
    const float* vl = v + static_cast<size_t>(l) * per;
    for (int t = 0; t < count; ++t)
      for (int h = 0; h < H; ++h)
        for (int c = 0; c < d; ++c) {
          const size_t src = (static_cast<size_t>(t) * H + h) * d + c;
          const size_t dst = (static_cast<size_t>(h) * count + t) * d + c;
          hk[dst] = to_bf16(kl[src]);
          hv[dst] = to_bf16(vl[src]);
        }
    cuda_check(cudaMemcpyAsync(dk, hk.data(), per * 2, cudaMemcpyHostToDevice, st(stream_)), "append_tokens");
    cuda_check(cudaMemcpyAsync(dv, hv.data(), per * 2, cudaMemcpyHostToDevice, st(stream_)), "append_tokens");
    check(sfi_append_block(&dev_->shape(), &dev_->cache(), l, count, dk, dv, stream_));
    cuda_check(cudaStreamSynchronize(st(stream_)), "append_tokens");
  }
  len_ += count;
}

std::vector<float> KvStore::key_row(int layer, Pos pos) const {
  if (pos < 1 || pos > len_) fail(ErrorCode::kOutOfRange, "KvStore: position " + std::to_string(pos) + " not written");
  const int H = spec_.n_kv_heads, d = spec_.head_dim;
  std::vector<uint16_t> raw(static_cast<size_t>(H) * d);
  const uint16_t* base = static_cast<const uint16_t*>(dev_->cache().k_cache);
  for (int h = 0; h < H; ++h) {
    const size_t off = ((static_cast<size_t>(layer) * H + h) * spec_.max_positions + (pos - 1)) * d;
    cuda_check(cudaMemcpy(raw.data() + static_cast<size_t>(h) * d, base + off, d * 2, cudaMemcpyDeviceToHost), "key_row");
  }
  std::vector<float> out(raw.size());
  for (size_t i = 0; i < raw.size(); ++i) out[i] = from_bf16(raw[i]);
  return out;
}

std::vector<float> KvStore::value_row(int layer, Pos pos) const {
  if (pos < 1 || pos > len_) fail(ErrorCode::kOutOfRange, "KvStore: position " + std::to_string(pos) + " not written");
  const int H = spec_.n_kv_heads, d = spec_.head_dim;
  std::vector<uint16_t> raw(static_cast<size_t>(H) * d);
  const uint16_t* base = static_cast<const uint16_t*>(dev_->cache().v_cache);
  for (int h = 0; h < H; ++h) {
    const size_t off = ((static_cast<size_t>(layer) * H + h) * spec_.max_positions + (pos - 1)) * d;
    cuda_check(cudaMemcpy(raw.data() + static_cast<size_t>(h) * d, base + off, d * 2, cudaMemcpyDeviceToHost), "value_row");
  }
  std::vector<float> out(raw.size());
  for (size_t i = 0; i < raw.size(); ++i) out[i] = from_bf16(raw[i]);
  return out;
}

double KvStore::key_norm(int layer, int head, Pos pos) const {
  if (pos < 1 || pos > len_)
    fail(ErrorCode::kOutOfRange, "KvStore: no key norm for position " + std::to_string(pos));
  double v = 0.0;
  const size_t off = (static_cast<size_t>(layer) * spec_.n_kv_heads + head) * spec_.max_positions + (pos - 1);
  cuda_check(cudaMemcpy(&v, dev_->cache().key_norms + off, 8, cudaMemcpyDeviceToHost), "key_norm");
  return v;
}

void KvStore::reorganize(int layer, const std::vector<Pos>& sink,
                         const std::vector<std::vector<Pos>>& selected) {
  // attention.cpp:186-217 checks, in order
  const int H = spec_.n_kv_heads;
  if (static_cast<int>(selected.size()) != H)
    fail(ErrorCode::kSupportMismatch, "reorganize: selected sets must cover every KV head");
  std::vector<std::vector<Pos>> merged(H);
  for (int h = 0; h < H; ++h) {
    std::merge(sink.begin(), sink.end(), selected[h].begin(), selected[h].end(), std::back_inserter(merged[h]));
    for (size_t i = 0; i + 1 < merged[h].size(); ++i)
      if (merged[h][i] >= merged[h][i + 1])
        fail(ErrorCode::kOverlapViolation, "reorganize: sink and selected sets overlap or are unsorted");
    for (Pos p : merged[h])
      if (p < 1 || p > len_) fail(ErrorCode::kOutOfRange, "reorganize: position " + std::to_string(p) + " not written");
  }
  // device layout: sink = positions 1..m stored ahead of the selected rows
  const int m = static_cast<int>(sink.size());
  for (int i = 0; i < m; ++i)
    if (sink[i] != i + 1)
      fail(ErrorCode::kUnsupported, "reorganize: the device compact layout needs sink = {1..n_sink}");
  if (m > limits_.n_sink) fail(ErrorCode::kUnsupported, "reorganize: sink larger than CacheLimits::n_sink");
  const int K = limits_.k_budget;
  std::vector<int32_t> sel(static_cast<size_t>(H) * std::max(K, 1), 0), cnt(H);
  for (int h = 0; h < H; ++h) {
    if (static_cast<int>(selected[h].size()) > K)
      fail(ErrorCode::kUnsupported, "reorganize: selected set larger than CacheLimits::k_budget");
    std::copy(selected[h].begin(), selected[h].end(), sel.begin() + static_cast<size_t>(h) * std::max(K, 1));
    cnt[h] = static_cast<int32_t>(selected[h].size());
  }
  set_window(m, 0);
  check(sfi_set_selection(&dev_->shape(), &dev_->cache(), layer, sel.data(), cnt.data(), stream_));
  uint32_t flags = 0;
  check(sfi_read_errors(&dev_->cache(), &flags, stream_));
  layers_[layer].positions = std::move(merged);
  layers_[layer].valid = true;
  layers_[layer].n_sink = m;
}

bool KvStore::compact_matches(int layer, const std::vector<Pos>& sink,
                              const std::vector<std::vector<Pos>>& selected) const {
  const LayerState& l = layers_[layer];
  if (!l.valid) return false;
  if (static_cast<int>(selected.size()) != spec_.n_kv_heads) return false;
  for (int h = 0; h < spec_.n_kv_heads; ++h) {
    std::vector<Pos> merged;
    std::merge(sink.begin(), sink.end(), selected[h].begin(), selected[h].end(), std::back_inserter(merged));
    if (merged != l.positions[h]) return false;
  }
  return true;
}

KvStore::CompactSegment KvStore::compact(int layer, int head) const {
  CompactSegment seg;
  const LayerState& l = layers_[layer];
  if (!l.valid) return seg;
  seg.positions = l.positions[head];
  const int d = spec_.head_dim;
  const size_t n = seg.positions.size();
  const int crows = limits_.n_recent + limits_.n_sink + limits_.k_budget;
  const size_t row0 = (static_cast<size_t>(layer) * spec_.n_kv_heads + head) * crows + limits_.n_recent;
  std::vector<uint16_t> rk(n * d), rv(n * d);
  if (n) {
    cuda_check(cudaMemcpy(rk.data(), static_cast<const uint16_t*>(dev_->cache().ck) + row0 * d, n * d * 2,
                          cudaMemcpyDeviceToHost), "compact");
    cuda_check(cudaMemcpy(rv.data(), static_cast<const uint16_t*>(dev_->cache().cv) + row0 * d, n * d * 2,
                          cudaMemcpyDeviceToHost), "compact");
  }
  seg.k.resize(n * d);
  seg.v.resize(n * d);
  for (size_t i = 0; i < n * d; ++i) {
    seg.k[i] = from_bf16(rk[i]);
    seg.v[i] = from_bf16(rv[i]);
  }
  return seg;
}

std::pair<Pos, int> KvStore::recent_tail(int n_recent) const {
  const int len = std::min<int>(n_recent, len_);
  return {len_ - len + 1, len};
}

// ---------------------------------------------------------------------------
// attention kernels

namespace {

struct DecodeIO {
  float* q;
  float* out;
};

DecodeIO stage_q(const KvStore& store, const std::vector<double>& q) {
  const ModelSpec& spec = store.spec();
  const size_t n = static_cast<size_t>(spec.n_query_heads) * spec.head_dim;
  if (q.size() != n) fail(ErrorCode::kSupportMismatch, "attention: q must hold n_query_heads * head_dim values");
  float* base = static_cast<float*>(t_scratch.get(al(n * 4) * 2));
  std::vector<float> qf(q.begin(), q.end());
  cuda_check(cudaMemcpyAsync(base, qf.data(), n * 4, cudaMemcpyHostToDevice, st(store.stream())), "attention");
  return {base, base + al(n * 4) / 4};
}

std::vector<double> fetch_out(const KvStore& store, const DecodeIO& io) {
  const ModelSpec& spec = store.spec();
  const size_t n = static_cast<size_t>(spec.n_query_heads) * spec.head_dim;
  std::vector<float> o(n);
  cuda_check(cudaMemcpyAsync(o.data(), io.out, n * 4, cudaMemcpyDeviceToHost, st(store.stream())), "attention");
  cuda_check(cudaStreamSynchronize(st(store.stream())), "attention");
  uint32_t flags = 0;
  check(sfi_read_errors(&store.device().cache(), &flags, store.stream()));
  return std::vector<double>(o.begin(), o.end());
}

}  // namespace

std::vector<double> attention_kernel_dense(const KvStore& store, int layer, const std::vector<double>& q,
                                           KernelStats* stats) {
  const ModelSpec& spec = store.spec();
  if (store.size() < 1) fail(ErrorCode::kOutOfRange, "KvStore: position 1 not written");
  store.set_window(0, 0);
  DecodeIO io = stage_q(store, q);
  check(sfi_dense_decode(&store.device().shape(), &store.device().cache(), layer, io.q, io.out, nullptr,
                         SFI_POOL_MEAN, store.stream()));
  std::vector<double> out = fetch_out(store, io);
  if (stats) {
    stats->reads += static_cast<std::uint64_t>(spec.n_kv_heads) * store.size();
    stats->flops += 2ull * store.size() * spec.head_dim * spec.n_query_heads;
  }
  return out;
}

std::vector<double> attention_kernel_sparse(const KvStore& store, int layer, const std::vector<double>& q,
                                            const SupportSet& support, KernelStats* stats) {
  const ModelSpec& spec = store.spec();
  if (!store.compact_matches(layer, support.sink, support.selected))
    fail(ErrorCode::kStaleCompact, "attention_kernel_sparse: compact buffer does not match the support");
  if (support.recent_len > 0) {
    if (support.recent_start < 1 || support.recent_start + support.recent_len - 1 > store.size())
      fail(ErrorCode::kOutOfRange, "KvStore: position " + std::to_string(support.recent_start) + " not written");
    if (support.recent_start + support.recent_len - 1 != store.size())
      fail(ErrorCode::kUnsupported, "attention_kernel_sparse: the device ring holds the tail ending at size()");
  }
  const int R = store.device().shape().n_recent;
  if (support.recent_len > R)
    fail(ErrorCode::kUnsupported, "attention_kernel_sparse: recent tail longer than the ring (n_recent)");
  std::uint64_t reads = 0;
  for (int h = 0; h < spec.n_kv_heads; ++h) {
    const int total = support.size_for_head(h);
    if (total == 0) fail(ErrorCode::kEmptySupport, "sparse_attention_step: empty support");
    reads += static_cast<std::uint64_t>(total);
  }
  store.set_window(static_cast<int>(support.sink.size()), support.recent_len);
  DecodeIO io = stage_q(store, q);
  check(sfi_sparse_decode(&store.device().shape(), &store.device().cache(), layer, io.q, io.out, store.stream()));
  std::vector<double> out = fetch_out(store, io);
  if (stats) {
    stats->reads += reads;
    for (int h = 0; h < spec.n_kv_heads; ++h)
      stats->flops += 2ull * support.size_for_head(h) * spec.head_dim * spec.group_size();
  }
  return out;
}

DenseCapture dense_capture(const KvStore& store, int layer, const std::vector<double>& q,
                           const std::vector<Pos>& allowed, PoolMode pool) {
  const ModelSpec& spec = store.spec();
  const Pos L = store.size();
  if (L < 1) fail(ErrorCode::kOutOfRange, "KvStore: position 1 not written");
  for (Pos j : allowed)
    if (j < 1 || j > L)
      fail(ErrorCode::kOutOfRange, "dense_attention_step: allowed position " + std::to_string(j) + " out of range");
  for (size_t i = 1; i < allowed.size(); ++i)
    if (allowed[i] != allowed[i - 1] + 1)
      fail(ErrorCode::kUnsupported, "dense_capture: J must be one contiguous range (decode J, scheduler.cpp:81-91)");
  const int nJ = static_cast<int>(allowed.size());
  const int nsb = nJ ? allowed.front() - 1 : 0;
  const int rl = nJ ? L - allowed.back() : 0;
  DenseCapture cap;
  cap.window.width = 1;
  cap.window.allowed = allowed;
  cap.window.values.assign(spec.n_kv_heads, std::vector<double>(nJ));
  // J = [n_sink_b + 1, L - recent_len] on the device
  store.set_window(nsb, rl);
  DecodeIO io = stage_q(store, q);
  float* logits = store.device().logits();
  check(sfi_dense_decode(&store.device().shape(), &store.device().cache(), layer, io.q, io.out,
                         nJ ? logits : nullptr, pool == PoolMode::kMax ? SFI_POOL_MAX : SFI_POOL_MEAN,
                         store.stream()));
  cap.context = fetch_out(store, io);
  if (nJ) {
    std::vector<float> lg(static_cast<size_t>(nJ));
    for (int h = 0; h < spec.n_kv_heads; ++h) {
      cuda_check(cudaMemcpy(lg.data(), logits + static_cast<size_t>(h) * spec.max_positions, nJ * 4,
                            cudaMemcpyDeviceToHost), "dense_capture");
      std::copy(lg.begin(), lg.end(), cap.window.values[h].begin());
    }
  }
  return cap;
}

// ---------------------------------------------------------------------------
// scheduler (scheduler.cpp:28-131): host-side integer bookkeeping

std::vector<Pos> SparseState::recent() const {
  std::vector<Pos> out(static_cast<size_t>(recent_len));
  std::iota(out.begin(), out.end(), recent_start);
  return out;
}

SupportSet SparseState::support() const {
  SupportSet s;
  s.sink = sink;
  s.selected = selected;
  s.recent_start = recent_start;
  s.recent_len = recent_len;
  return s;
}

namespace {

void slide(SparseState& s, Pos prefix_len, const CacheLimits& limits) {
  int32_t rs = 0, rl = 0;
  sfi_recent_window(prefix_len, static_cast<int32_t>(s.sink.size()), limits.n_recent, &rs, &rl);
  s.recent_len = rl;
  s.recent_start = rs;
}

bool in_recent(const SparseState& s, Pos p) { return p >= s.recent_start && p < s.recent_start + s.recent_len; }

}  // namespace

DecodeState init_decode_state(Pos prompt_len, int n_layers, int n_kv_heads, const CacheLimits& limits) {
  limits.validate();
  if (prompt_len < 1) fail(ErrorCode::kOutOfRange, "init_decode_state: empty prompt");
  DecodeState state;
  state.prefix_len = prompt_len;
  state.g = 1;
  state.per_layer.resize(static_cast<size_t>(n_layers));
  const int n_sink = std::min<int>(limits.n_sink, prompt_len);
  for (int l = 0; l < n_layers; ++l) {
    SparseState& s = state.per_layer[l];
    s.layer = l;
    s.sink.resize(static_cast<size_t>(n_sink));
    std::iota(s.sink.begin(), s.sink.end(), Pos{1});
    s.selected.assign(static_cast<size_t>(n_kv_heads), {});
    slide(s, prompt_len, limits);
  }
  return state;
}

std::vector<Pos> compute_allowed(const SparseState& state, Pos prefix_len) {
  if (prefix_len < 1) fail(ErrorCode::kOutOfRange, "compute_allowed: prefix_len must be >= 1");
  std::vector<Pos> out;
  for (Pos p = 1; p <= prefix_len; ++p) {
    if (std::binary_search(state.sink.begin(), state.sink.end(), p)) continue;
    if (in_recent(state, p)) continue;
    out.push_back(p);
  }
  return out;
}

int next_step_type(const DecodeState& state, const TriggerConfig& trig) {
  if (trig.is_trigger(state.last_token)) return 1;
  if (state.steps_since_slow + 1 >= trig.t_max) return 1;
  return 0;
}

void fast_step_update(DecodeState& state, const CacheLimits& limits) {
  state.t += 1;
  state.prefix_len += 1;
  state.steps_since_slow += 1;
  for (SparseState& s : state.per_layer) slide(s, state.prefix_len, limits);
}

void slow_step_update(DecodeState& state, const std::vector<std::vector<std::vector<Pos>>>& selected_per_layer,
                      const CacheLimits& limits) {
  if (selected_per_layer.size() != state.per_layer.size())
    fail(ErrorCode::kSupportMismatch, "slow_step_update: one selected set per layer required");
  for (size_t l = 0; l < state.per_layer.size(); ++l) {
    SparseState& s = state.per_layer[l];
    for (const std::vector<Pos>& head_sel : selected_per_layer[l]) {
      if (static_cast<int>(head_sel.size()) > limits.k_budget)
        fail(ErrorCode::kOutOfRange, "slow_step_update: selected set exceeds k_budget");
      for (Pos p : head_sel)
        if (std::binary_search(s.sink.begin(), s.sink.end(), p) || in_recent(s, p))
          fail(ErrorCode::kOverlapViolation,
               "slow_step_update: selected position " + std::to_string(p) + " overlaps sink or recent");
    }
    s.selected = selected_per_layer[l];
  }
  state.t += 1;
  state.prefix_len += 1;
  state.steps_since_slow = 0;
  for (SparseState& s : state.per_layer) slide(s, state.prefix_len, limits);
}

double flop_model(double prefix_len, double support, double slow_fraction) {
  if (!(support > 0.0) || support > prefix_len)
    fail(ErrorCode::kOutOfRange, "flop_model: support must be in (0, L]");
  if (slow_fraction < 0.0 || slow_fraction > 1.0)
    fail(ErrorCode::kOutOfRange, "flop_model: slow_fraction must be in [0, 1]");
  const double mixed = slow_fraction * prefix_len + (1.0 - slow_fraction) * support;
  return prefix_len / mixed;
}

}  // namespace sfi_b200

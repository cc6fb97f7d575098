// engine.cpp — END-TO-END TEST HARNESS (harness/sfi_toy.hpp, libsfi_toy.so;
// not in the product library): the reference's request loop around the device
// hot path.
//
//   run_request     scheduler.cpp:213-330   prefill + slow/fast decode loop
//   run_dense       scheduler.cpp:332-365   dense greedy baseline
//   run_step        attention.cpp:303-440   one token through every layer
//   prefill_dense   attention.cpp:460-500   tail-window capture over frozen J
//   ToyModel        model.cpp:36-167        weights (same RNG draws)
//
// Host fp64 here: the toy decoder's embedding, RMSNorm, projections, RoPE, MLP
// and LM head, in the reference's operation order (the oracle build's
// sequential dot products), plus the scheduler bookkeeping. Device: every KV
// append (paged rows, recent ring, key norms), dense attention with the
// pooled-logit capture (K1), the cache-mode Selector (K2, also the W-row
// prefill window), the compact rebuild (K3) and the sparse attention (K4) —
// the same entry points the batched production path launches.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <random>

#include "sfi_b200.hpp"
#include "sfi_toy.hpp"

namespace sfi {

namespace {

constexpr double kNormEps = 1e-6;  // attention.cpp:28

void cuda_ok(cudaError_t e, const char* what) {
  if (e != cudaSuccess) fail(ErrorCode::kCuda, std::string(what) + ": " + cudaGetErrorString(e));
}

// Grow-only device staging owned by the calling thread.
struct Staging {
  void* p = nullptr;
  size_t n = 0;
  void* get(size_t bytes) {
    if (bytes > n) {
      if (p) cudaFree(p);
      p = nullptr;
      n = 0;
      cuda_ok(cudaMalloc(&p, bytes), "engine staging");
      n = bytes;
    }
    return p;
  }
  ~Staging() {
    if (p) cudaFree(p);
  }
};
thread_local Staging t_stage;

size_t al(size_t x) { return (x + 255) & ~size_t(255); }

// model.cpp:36-44: drawn in double, rounded to fp32, held as double; one
// distribution object per matrix, rows then columns.
ToyModel::Matrix random_matrix(int rows, int cols, double stddev, std::mt19937_64& rng) {
  std::normal_distribution<double> dist(0.0, stddev);
  ToyModel::Matrix m;
  m.rows = rows;
  m.cols = cols;
  m.v.resize(static_cast<size_t>(rows) * cols);
  for (int r = 0; r < rows; ++r)
    for (int c = 0; c < cols; ++c) m.v[static_cast<size_t>(r) * cols + c] = static_cast<double>(static_cast<float>(dist(rng)));
  return m;
}

std::vector<double> matvec(const ToyModel::Matrix& m, const double* x) {
  std::vector<double> out(static_cast<size_t>(m.rows));
  for (int r = 0; r < m.rows; ++r) {
    const double* row = m.row(r);
    double acc = 0.0;
    for (int c = 0; c < m.cols; ++c) acc += row[c] * x[c];
    out[r] = acc;
  }
  return out;
}

// attention.cpp:30-34
std::vector<double> rmsnorm(const std::vector<double>& x, const std::vector<double>& g) {
  double ss = 0.0;
  for (double v : x) ss += v * v;
  const double ms = ss / static_cast<double>(x.size());
  const double inv = 1.0 / std::sqrt(ms + kNormEps);
  std::vector<double> out(x.size());
  for (size_t i = 0; i < x.size(); ++i) out[i] = x[i] * inv * g[i];
  return out;
}

double silu(double x) { return x / (1.0 + std::exp(-x)); }  // attention.cpp:36

// attention.cpp:38-54: pairs (2i, 2i+1), 0-based position angle.
void apply_rope(double* vec, int n_heads, int d, Pos pos, double base) {
  const double p = static_cast<double>(pos - 1);
  for (int h = 0; h < n_heads; ++h) {
    double* head = vec + static_cast<std::ptrdiff_t>(h) * d;
    for (int i = 0; i < d / 2; ++i) {
      const double theta = p * std::pow(base, -2.0 * i / d);
      const double c = std::cos(theta);
      const double s = std::sin(theta);
      const double a = head[2 * i];
      const double b = head[2 * i + 1];
      head[2 * i] = a * c - b * s;
      head[2 * i + 1] = a * s + b * c;
    }
  }
}

// One contiguous J = [lo, hi] restricted to positions <= pos (prefill rows
// capture against a frozen J and mask what they cannot reach).
struct JRange {
  Pos lo = 1, hi = 0;
  int size() const { return hi >= lo ? hi - lo + 1 : 0; }
};
JRange contiguous_j(const std::vector<Pos>& allowed, Pos pos) {
  JRange r;
  if (allowed.empty()) return r;
  for (size_t i = 1; i < allowed.size(); ++i)
    if (allowed[i] != allowed[i - 1] + 1)
      fail(ErrorCode::kUnsupported, "capture: J must be one contiguous range (decode / prefill J)");
  r.lo = allowed.front();
  r.hi = std::min<Pos>(allowed.back(), pos);
  return r;
}

struct StepMode {
  const CaptureSpec* capture = nullptr;
  const std::vector<SupportSet>* support = nullptr;  // sparse when set
  bool compute_logits = true;
  bool allow_forward_mask = false;
  // Slow decode step: run the cache-mode Selector after each layer's capture
  // and return the per-layer selections (refresh_selected, scheduler.cpp:
  // 162-180, with the same per-layer inputs).
  const SelectorConfig* select = nullptr;
  std::vector<std::vector<std::vector<Pos>>>* selected = nullptr;
  // Prefill: keep the post-RoPE q of the tail rows, fp32 [n_layers][Hq*d].
  std::vector<std::vector<float>>* keep_q = nullptr;
};

std::vector<std::vector<Pos>> read_selection(const KvStore& store, int layer) {
  const sfi_cache& c = store.device().cache();
  const sfi_shape& s = store.device().shape();
  const int H = s.n_kv_heads, K = std::max(s.k_budget, 1);
  std::vector<int32_t> cnt(H), sel(static_cast<size_t>(H) * K);
  cuda_ok(cudaStreamSynchronize(static_cast<cudaStream_t>(store.stream())), "selection");
  cuda_ok(cudaMemcpy(cnt.data(), c.n_sel + static_cast<size_t>(layer) * H, H * 4, cudaMemcpyDeviceToHost),
          "selection");
  cuda_ok(cudaMemcpy(sel.data(), c.sel + static_cast<size_t>(layer) * H * K, sel.size() * 4, cudaMemcpyDeviceToHost),
          "selection");
  std::vector<std::vector<Pos>> out(static_cast<size_t>(H));
  for (int h = 0; h < H; ++h)
    out[h].assign(sel.begin() + static_cast<size_t>(h) * K, sel.begin() + static_cast<size_t>(h) * K + cnt[h]);
  return out;
}

void read_errors(const KvStore& store) {
  uint32_t flags = 0;
  check(sfi_read_errors(&store.device().cache(), &flags, store.stream()));
}

StepOutput run_step(const ToyModel& model, TokenId token, KvStore& store, const StepMode& mode) {
  const ModelSpec& spec = model.spec();
  if (token < 0 || token >= spec.vocab_size) fail(ErrorCode::kOutOfRange, "step: token id out of range");
  const bool sparse = mode.support != nullptr;
  const CaptureSpec* cap = mode.capture;
  const int d = spec.head_dim, hq = spec.n_query_heads, hk = spec.n_kv_heads, group = spec.group_size();

  store.begin_token();
  const Pos pos = store.size() + 1;
  if (cap != nullptr && cap->window) {
    for (Pos j : cap->allowed)
      if (j < 1 || (j > pos && !mode.allow_forward_mask))
        fail(ErrorCode::kOutOfRange, "dense_attention_step: allowed position " + std::to_string(j) + " out of range");
  }
  if (sparse) {
    if (static_cast<int>(mode.support->size()) != spec.n_layers)
      fail(ErrorCode::kSupportMismatch, "sparse_attention_step: one support per layer required");
    for (const SupportSet& s : *mode.support) {
      if (s.recent_len > 0 && s.recent_start + s.recent_len - 1 != pos)
        fail(ErrorCode::kOutOfRange, "sparse_attention_step: recent tail must end at the current position");
      if (s.recent_len == 0 && !std::binary_search(s.sink.begin(), s.sink.end(), pos))
        fail(ErrorCode::kOutOfRange, "sparse_attention_step: current position not in support");
    }
  }
  if (mode.select && mode.select->k_budget != store.limits().k_budget)
    fail(ErrorCode::kUnsupported, "run_request: SelectorConfig::k_budget must equal CacheLimits::k_budget");

  StepOutput out;
  const bool window = cap != nullptr && cap->window;
  if (window) out.attn_logits.emplace();
  const JRange J = window ? contiguous_j(cap->allowed, pos) : JRange{};
  const int nJ = J.size();
  if (mode.selected) mode.selected->assign(static_cast<size_t>(spec.n_layers), {});

  const sfi_shape& dshape = store.device().shape();
  const sfi_cache& dcache = store.device().cache();
  cudaStream_t stream = static_cast<cudaStream_t>(store.stream());
  const size_t nq = static_cast<size_t>(hq) * d;
  float* dq = static_cast<float*>(t_stage.get(al(nq * 4) * 2));
  float* dout = dq + al(nq * 4) / 4;
  std::vector<float> qf(nq), of(nq);
  std::vector<float> lg;

  const ToyModel::Matrix& E = model.embedding();
  std::vector<double> h(E.row(token), E.row(token) + E.cols);
  for (int l = 0; l < spec.n_layers; ++l) {
    const ToyModel::LayerWeights& lw = model.layer(l);
    const std::vector<double> a = rmsnorm(h, lw.ln1);
    std::vector<double> q = matvec(lw.wq, a.data());
    std::vector<double> k = matvec(lw.wk, a.data());
    const std::vector<double> v = matvec(lw.wv, a.data());
    apply_rope(q.data(), hq, d, pos, spec.rope_base);
    apply_rope(k.data(), hk, d, pos, spec.rope_base);
    std::vector<float> kf(static_cast<size_t>(hk) * d), vf(static_cast<size_t>(hk) * d);
    for (int i = 0; i < hk * d; ++i) {
      kf[i] = static_cast<float>(k[i]);
      vf[i] = static_cast<float>(v[i]);
    }
    store.append_layer(l, kf.data(), vf.data());  // paged row, ring slot, fp64 norm (device)
    if (sparse && !store.compact_matches(l, (*mode.support)[l].sink, (*mode.support)[l].selected))
      fail(ErrorCode::kStaleCompact, "sparse_attention_step: compact buffer does not match the requested support");
    for (size_t i = 0; i < nq; ++i) qf[i] = static_cast<float>(q[i]);
    if (mode.keep_q) (*mode.keep_q)[l] = qf;
    cuda_ok(cudaMemcpyAsync(dq, qf.data(), nq * 4, cudaMemcpyHostToDevice, stream), "step q");

    if (sparse) {
      const SupportSet& sup = (*mode.support)[l];
      for (int hh = 0; hh < hk; ++hh) {
        const int total = sup.size_for_head(hh);
        if (total == 0) fail(ErrorCode::kEmptySupport, "sparse_attention_step: empty support");
        out.kv_read_count += static_cast<std::uint64_t>(total);
        out.flop_count += 2ull * static_cast<std::uint64_t>(total) * d * group;
      }
      store.set_window(static_cast<int>(sup.sink.size()), sup.recent_len, pos);
      check(sfi_sparse_decode(&dshape, &dcache, l, dq, dout, stream));
    } else {
      // J on the device = [n_sink_b + 1, L - recent_len]
      if (nJ > 0) store.set_window(J.lo - 1, pos - J.hi, pos);
      else store.set_window(0, 0, pos);
      out.kv_read_count += static_cast<std::uint64_t>(hk) * pos;
      out.flop_count += 2ull * static_cast<std::uint64_t>(pos) * d * hq;
      float* logits = nJ > 0 ? store.device().logits() : nullptr;
      const int pool = (cap && cap->pool == PoolMode::kMax) ? SFI_POOL_MAX : SFI_POOL_MEAN;
      check(sfi_dense_decode(&dshape, &dcache, l, dq, dout, logits, pool, stream));
      if (window) {
        LogitWindow w;
        w.width = 1;
        w.allowed = cap->allowed;
        w.values.assign(hk, std::vector<double>(cap->allowed.size(), kMaskedLogit));  // j > pos stay masked
        if (nJ > 0) {
          lg.resize(static_cast<size_t>(nJ));
          cuda_ok(cudaStreamSynchronize(stream), "capture");
          const size_t c0 = static_cast<size_t>(J.lo - cap->allowed.front());
          for (int hh = 0; hh < hk; ++hh) {
            cuda_ok(cudaMemcpy(lg.data(), logits + static_cast<size_t>(hh) * spec.max_positions, nJ * 4,
                               cudaMemcpyDeviceToHost), "capture");
            for (int c = 0; c < nJ; ++c) w.values[hh][c0 + c] = lg[c];
          }
        }
        out.attn_logits->push_back(std::move(w));
      }
      if (mode.select) {
        // refresh_selected for this layer: J empty -> nothing to select
        if (nJ > 0 && static_cast<int>(cap->allowed.size()) == nJ) {
          const sfi_selector_params prm = to_params(*mode.select);
          check(sfi_selector(&dshape, &dcache, l, logits, &prm, stream));
          read_errors(store);
          (*mode.selected)[l] = read_selection(store, l);
        } else {
          (*mode.selected)[l].assign(static_cast<size_t>(hk), {});
        }
      }
    }
    cuda_ok(cudaMemcpyAsync(of.data(), dout, nq * 4, cudaMemcpyDeviceToHost, stream), "step out");
    cuda_ok(cudaStreamSynchronize(stream), "step out");
    read_errors(store);
    std::vector<double> ctx(of.begin(), of.end());
    const std::vector<double> o = matvec(lw.wo, ctx.data());
    for (size_t i = 0; i < h.size(); ++i) h[i] += o[i];
    const std::vector<double> bn = rmsnorm(h, lw.ln2);
    const std::vector<double> gate = matvec(lw.w_gate, bn.data());
    const std::vector<double> up = matvec(lw.w_up, bn.data());
    std::vector<double> act(gate.size());
    for (size_t i = 0; i < gate.size(); ++i) act[i] = silu(gate[i]) * up[i];
    const std::vector<double> down = matvec(lw.w_down, act.data());
    for (size_t i = 0; i < h.size(); ++i) h[i] += down[i];
  }
  store.end_token();
  if (mode.compute_logits) {
    const std::vector<double> hf = rmsnorm(h, model.final_norm());
    std::vector<double> logits = matvec(model.lm_head(), hf.data());
    for (size_t i = 0; i < logits.size(); ++i) logits[i] += model.lm_bias()[i];
    out.vocab_logits = std::move(logits);
  }
  return out;
}

// prefill_dense with the tail rows' q kept; returns the row count and the
// per-layer q of those rows ([n_layers][rows][Hq*d] fp32).
int prefill_rows(const ToyModel& model, const std::vector<TokenId>& tokens, KvStore& store, int window_width,
                 const std::vector<Pos>& allowed, std::vector<std::vector<std::vector<float>>>& q_rows) {
  const ModelSpec& spec = model.spec();
  const int n = static_cast<int>(tokens.size());
  int rows = std::min(window_width, n);
  if (!allowed.empty()) rows = std::min(rows, n - allowed.front() + 1);
  rows = std::max(rows, 0);
  q_rows.assign(static_cast<size_t>(spec.n_layers), std::vector<std::vector<float>>(static_cast<size_t>(rows)));
  std::vector<std::vector<float>> keep(static_cast<size_t>(spec.n_layers));
  for (int i = 0; i < n; ++i) {
    const bool tail = i >= n - rows;
    StepMode mode;
    mode.compute_logits = false;
    mode.allow_forward_mask = true;
    mode.keep_q = tail ? &keep : nullptr;
    run_step(model, tokens[i], store, mode);
    if (tail)
      for (int l = 0; l < spec.n_layers; ++l) q_rows[l][i - (n - rows)] = keep[l];
  }
  return rows;
}

// Pooled tail-window logits of one layer on the device (sfi_prefill_capture),
// J = allowed (contiguous, inside the written prefix); returns the device
// buffer [H][rows][max_positions].
float* capture_window(const KvStore& store, int layer, const std::vector<std::vector<float>>& q_rows,
                      const std::vector<Pos>& allowed, Pos first_row_pos, PoolMode pool) {
  const ModelSpec& spec = store.spec();
  const int rows = static_cast<int>(q_rows.size());
  const size_t nq = static_cast<size_t>(spec.n_query_heads) * spec.head_dim;
  const size_t b_q = al(rows * nq * 4), b_p = al(rows * 4);
  const size_t b_out = al(static_cast<size_t>(spec.n_kv_heads) * rows * spec.max_positions * 4);
  uint8_t* base = static_cast<uint8_t*>(t_stage.get(b_q + b_p + b_out));
  float* dq = reinterpret_cast<float*>(base);
  int32_t* dpos = reinterpret_cast<int32_t*>(base + b_q);
  float* dout = reinterpret_cast<float*>(base + b_q + b_p);
  std::vector<float> q(rows * nq);
  std::vector<int32_t> qp(rows);
  for (int r = 0; r < rows; ++r) {
    std::copy(q_rows[r].begin(), q_rows[r].end(), q.begin() + r * nq);
    qp[r] = first_row_pos + r;
  }
  cudaStream_t stream = static_cast<cudaStream_t>(store.stream());
  cuda_ok(cudaMemcpyAsync(dq, q.data(), q.size() * 4, cudaMemcpyHostToDevice, stream), "prefill capture");
  cuda_ok(cudaMemcpyAsync(dpos, qp.data(), rows * 4, cudaMemcpyHostToDevice, stream), "prefill capture");
  store.set_window(allowed.front() - 1, store.size() - allowed.back());
  check(sfi_prefill_capture(&store.device().shape(), &store.device().cache(), layer, dq, rows, dpos, dout,
                            pool == PoolMode::kMax ? SFI_POOL_MAX : SFI_POOL_MEAN, stream));
  return dout;
}

}  // namespace

ToyModel ToyModel::random(const ModelSpec& spec, std::uint64_t seed) {
  spec.validate();
  ToyModel m;
  m.spec_ = spec;
  std::mt19937_64 rng(seed);
  const int hidden = spec.hidden(), ff = spec.ff_dim();
  const double w_std = 1.0 / std::sqrt(static_cast<double>(hidden));
  const double ff_std = 1.0 / std::sqrt(static_cast<double>(ff));
  m.embed_ = random_matrix(spec.vocab_size, hidden, 1.0, rng);
  m.layers_.resize(static_cast<size_t>(spec.n_layers));
  for (auto& lw : m.layers_) {
    lw.ln1.assign(static_cast<size_t>(hidden), 1.0);
    lw.wq = random_matrix(spec.n_query_heads * spec.head_dim, hidden, w_std, rng);
    lw.wk = random_matrix(spec.n_kv_heads * spec.head_dim, hidden, w_std, rng);
    lw.wv = random_matrix(spec.n_kv_heads * spec.head_dim, hidden, w_std, rng);
    lw.wo = random_matrix(hidden, spec.n_query_heads * spec.head_dim, w_std, rng);
    lw.ln2.assign(static_cast<size_t>(hidden), 1.0);
    lw.w_gate = random_matrix(ff, hidden, w_std, rng);
    lw.w_up = random_matrix(ff, hidden, w_std, rng);
    lw.w_down = random_matrix(hidden, ff, ff_std, rng);
  }
  m.ln_f_.assign(static_cast<size_t>(hidden), 1.0);
  m.lm_head_ = random_matrix(spec.vocab_size, hidden, w_std, rng);
  m.lm_bias_.assign(static_cast<size_t>(spec.vocab_size), 0.0);
  return m;
}

TokenId argmax_token(const std::vector<double>& logits) {  // attention.cpp:249-254
  int best = 0;
  for (int i = 1; i < static_cast<int>(logits.size()); ++i)
    if (logits[i] > logits[best]) best = i;
  return best;
}

StepOutput dense_attention_step(const ToyModel& model, TokenId token, KvStore& store, const CaptureSpec& capture) {
  StepMode mode;
  mode.capture = &capture;
  return run_step(model, token, store, mode);
}

StepOutput sparse_attention_step(const ToyModel& model, TokenId token, KvStore& store,
                                 const std::vector<SupportSet>& support) {
  StepMode mode;
  mode.support = &support;
  return run_step(model, token, store, mode);
}

std::vector<LogitWindow> prefill_dense(const ToyModel& model, const std::vector<TokenId>& tokens, KvStore& store,
                                       int window_width, const std::vector<Pos>& allowed, PoolMode pool) {
  const ModelSpec& spec = model.spec();
  const Pos start = store.size();
  std::vector<std::vector<std::vector<float>>> q_rows;
  const int rows = prefill_rows(model, tokens, store, window_width, allowed, q_rows);
  const int n = static_cast<int>(tokens.size());
  std::vector<LogitWindow> windows(static_cast<size_t>(spec.n_layers));
  for (auto& w : windows) {
    w.width = rows;
    w.allowed = allowed;
    w.values.assign(spec.n_kv_heads, std::vector<double>(static_cast<size_t>(rows) * allowed.size()));
  }
  if (rows == 0 || allowed.empty()) return windows;
  contiguous_j(allowed, store.size());
  if (allowed.back() > store.size()) fail(ErrorCode::kUnsupported, "prefill_dense: J must lie inside the prefix");
  const size_t nJ = allowed.size();
  std::vector<float> lg(nJ);
  for (int l = 0; l < spec.n_layers; ++l) {
    float* d = capture_window(store, l, q_rows[l], allowed, start + n - rows + 1, pool);
    cuda_ok(cudaStreamSynchronize(static_cast<cudaStream_t>(store.stream())), "prefill capture");
    read_errors(store);
    for (int hh = 0; hh < spec.n_kv_heads; ++hh)
      for (int r = 0; r < rows; ++r) {
        cuda_ok(cudaMemcpy(lg.data(), d + (static_cast<size_t>(hh) * rows + r) * spec.max_positions, nJ * 4,
                           cudaMemcpyDeviceToHost), "prefill capture");
        std::copy(lg.begin(), lg.end(), windows[l].values[hh].begin() + static_cast<size_t>(r) * nJ);
      }
  }
  return windows;
}

RequestResult run_request(const ToyModel& model, const std::vector<TokenId>& prompt, const CacheLimits& limits,
                          const TriggerConfig& trig, const SelectorConfig& cfg, int max_new,
                          const RunOptions& opts) {
  limits.validate();
  trig.validate();
  cfg.validate();
  if (prompt.empty()) fail(ErrorCode::kOutOfRange, "run_request: empty prompt");
  if (max_new < 1) fail(ErrorCode::kOutOfRange, "run_request: max_new must be >= 1");
  const ModelSpec& spec = model.spec();
  const Pos prompt_len = static_cast<Pos>(prompt.size());
  if (prompt_len + max_new > spec.max_positions)
    fail(ErrorCode::kContextOverflow, "run_request: prompt plus max_new exceeds max_positions");
  if (limits.n_sink + limits.n_recent > spec.max_positions)
    fail(ErrorCode::kConfig, "run_request: n_sink + n_recent exceeds the maximum context length");
  if (cfg.k_budget != limits.k_budget)
    fail(ErrorCode::kUnsupported, "run_request: SelectorConfig::k_budget must equal CacheLimits::k_budget");

  KvStore store(spec, limits);
  DecodeState state = init_decode_state(prompt_len, spec.n_layers, spec.n_kv_heads, limits);
  const std::vector<Pos> sink = state.per_layer[0].sink;
  RequestResult result;

  // prefill: dense pass over the prompt minus its last token, then the W-row
  // tail window through the device Selector (refresh_selected)
  if (prompt_len > 1) {
    const std::vector<TokenId> block(prompt.begin(), prompt.end() - 1);
    SparseState view = state.per_layer[0];
    const int rl = std::clamp<int>(static_cast<int>(prompt_len - 1) - static_cast<int>(view.sink.size()), 0,
                                   limits.n_recent);
    view.recent_len = rl;
    view.recent_start = prompt_len - 1 - rl + 1;
    const std::vector<Pos> allowed = compute_allowed(view, prompt_len - 1);
    std::vector<std::vector<std::vector<float>>> q_rows;
    const int rows = prefill_rows(model, block, store, trig.window_prefill, allowed, q_rows);
    for (int l = 0; l < spec.n_layers; ++l) {
      if (allowed.empty() || rows == 0) {
        state.per_layer[l].selected.assign(static_cast<size_t>(spec.n_kv_heads), {});
        continue;
      }
      float* d = capture_window(store, l, q_rows[l], allowed, prompt_len - 1 - rows + 1, cfg.pool);
      const sfi_selector_params prm = to_params(cfg);
      check(sfi_selector_window(&store.device().shape(), &store.device().cache(), l, d, rows, &prm, store.stream()));
      read_errors(store);
      state.per_layer[l].selected = read_selection(store, l);
    }
  }

  TokenId pending = prompt.back();
  std::vector<std::vector<std::vector<Pos>>> frozen(static_cast<size_t>(spec.n_layers));
  for (int l = 0; l < spec.n_layers; ++l) frozen[l] = state.per_layer[l].selected;

  for (int step = 0; step < max_new; ++step) {
    StepRecord rec;
    rec.t = step;
    rec.prefix_len = state.prefix_len;
    StepOutput out;
    if (state.g == 1) {
      rec.slow = true;
      rec.cause = step == 0 ? StepCause::kInitial
                  : trig.is_trigger(state.last_token) ? StepCause::kTrigger
                                                      : StepCause::kForced;
      CaptureSpec cap;
      cap.window = true;
      cap.allowed = compute_allowed(state.per_layer[0], state.prefix_len);
      cap.pool = cfg.pool;
      std::vector<std::vector<std::vector<Pos>>> selected;
      StepMode mode;
      mode.capture = &cap;
      mode.select = &cfg;
      mode.selected = &selected;
      out = run_step(model, pending, store, mode);
      rec.support_size = static_cast<int>(state.prefix_len);
      rec.allowed_size = static_cast<int>(cap.allowed.size());
      const TokenId token = argmax_token(out.vocab_logits);
      state.last_token = token;
      slow_step_update(state, selected, limits);
      for (int l = 0; l < spec.n_layers; ++l) {
        store.reorganize(l, sink, state.per_layer[l].selected);  // K3 on the device
        frozen[l] = state.per_layer[l].selected;
      }
      result.tokens.push_back(token);
    } else {
      std::vector<SupportSet> support(static_cast<size_t>(spec.n_layers));
      for (int l = 0; l < spec.n_layers; ++l) {
        if (state.per_layer[l].selected != frozen[l])
          fail(ErrorCode::kOverlapViolation, "run_request: selected memory mutated during a fast segment");
        support[l] = state.per_layer[l].support();
      }
      out = sparse_attention_step(model, pending, store, support);
      rec.support_size = support[0].size_for_head(0);
      result.fast_retention.push_back(static_cast<double>(rec.support_size) / static_cast<double>(state.prefix_len));
      const TokenId token = argmax_token(out.vocab_logits);
      state.last_token = token;
      fast_step_update(state, limits);
      result.tokens.push_back(token);
    }
    result.total_flops += out.flop_count;
    result.total_kv_reads += out.kv_read_count;
    result.dense_equiv_reads += static_cast<std::uint64_t>(spec.n_layers) * spec.n_kv_heads * rec.prefix_len;
    if (opts.collect_logits) result.step_logits.push_back(std::move(out.vocab_logits));
    if (opts.capture_selected) {
      std::vector<std::vector<std::vector<Pos>>> snap(static_cast<size_t>(spec.n_layers));
      for (int l = 0; l < spec.n_layers; ++l) snap[l] = state.per_layer[l].selected;
      result.selected_per_step.push_back(std::move(snap));
    }
    result.log.push_back(rec);
    pending = result.tokens.back();
    state.g = next_step_type(state, trig);
  }
  return result;
}

DenseResult run_dense(const ToyModel& model, const std::vector<TokenId>& prompt, int max_new) {
  if (prompt.empty()) fail(ErrorCode::kOutOfRange, "run_dense: empty prompt");
  if (max_new < 1) fail(ErrorCode::kOutOfRange, "run_dense: max_new must be >= 1");
  const ModelSpec& spec = model.spec();
  if (static_cast<Pos>(prompt.size()) + max_new > spec.max_positions)
    fail(ErrorCode::kContextOverflow, "run_dense: prompt plus max_new exceeds max_positions");
  KvStore store(spec);
  if (prompt.size() > 1) {
    const std::vector<TokenId> block(prompt.begin(), prompt.end() - 1);
    std::vector<std::vector<std::vector<float>>> q_rows;
    prefill_rows(model, block, store, 1, {}, q_rows);
  }
  DenseResult result;
  TokenId pending = prompt.back();
  for (int step = 0; step < max_new; ++step) {
    const StepOutput out = dense_attention_step(model, pending, store, CaptureSpec{});
    const TokenId token = argmax_token(out.vocab_logits);
    result.tokens.push_back(token);
    result.total_kv_reads += out.kv_read_count;
    result.total_flops += out.flop_count;
    result.step_logits.push_back(out.vocab_logits);
    pending = token;
  }
  return result;
}

}  // namespace sfi

// ref_capi.cpp — C-ABI wrapper over the UNMODIFIED reference library.
// TEST INFRASTRUCTURE ONLY: compiled by oracle/Makefile together with
// /root/reference/proj/src/*.cpp into oracle/_ref/libsfi_ref.so. Nothing in
// here re-implements reference arithmetic; every call forwards to the
// reference's own functions (namespace sfi).
#include <cmath>
#include <cstring>
#include <exception>
#include <memory>
#include <string>
#include <vector>

#include "oracle_abi.h"
#include "sfi/attention.hpp"
#include "sfi/config.hpp"
#include "sfi/error.hpp"
#include "sfi/scheduler.hpp"
#include "sfi/selector.hpp"

namespace {

void set_err(char* err, int errlen, const char* msg) {
  if (err && errlen > 0) {
    std::strncpy(err, msg, static_cast<std::size_t>(errlen) - 1);
    err[errlen - 1] = '\0';
  }
}

template <typename F>
int guarded(char* err, int errlen, F&& fn) {
  try {
    fn();
    return 0;
  } catch (const sfi::Error& e) {
    set_err(err, errlen, e.what());
    return 1 + static_cast<int>(e.code());
  } catch (const std::exception& e) {
    set_err(err, errlen, e.what());
    return 200;
  }
}

sfi::SelectorConfig to_cfg(const orc_selector_cfg* c) {
  sfi::SelectorConfig cfg;
  cfg.alpha = c->alpha;
  cfg.gamma = c->gamma;
  cfg.beta = c->beta;
  cfg.p_curve = c->p_curve;
  cfg.eta = c->eta;
  cfg.lambda_clip = c->lambda_clip;
  cfg.alpha_soft = c->alpha_soft;
  cfg.alpha_cross = c->alpha_cross;
  cfg.temperature = c->temperature;
  cfg.epsilon = c->epsilon;
  cfg.nms_radius = c->nms_radius;
  cfg.k_budget = c->k_budget;
  cfg.pool = c->pool == 1 ? sfi::PoolMode::kMax : sfi::PoolMode::kMean;
  return cfg;
}

struct StoreBox {
  sfi::ModelSpec spec;
  std::unique_ptr<sfi::KvStore> store;
};

std::vector<std::vector<sfi::Pos>> unflatten(int heads, const int32_t* counts,
                                             const int32_t* flat) {
  std::vector<std::vector<sfi::Pos>> out(static_cast<std::size_t>(heads));
  std::size_t off = 0;
  for (int h = 0; h < heads; ++h) {
    out[h].assign(flat + off, flat + off + counts[h]);
    off += static_cast<std::size_t>(counts[h]);
  }
  return out;
}

}  // namespace

extern "C" {

const char* orc_kind(void) { return "reference"; }

int orc_run_selector(int H, int W, int n, const int32_t* allowed,
                     const double* values, const double* norms,
                     const orc_selector_cfg* c, int32_t* out_sel, int out_cap,
                     int32_t* out_count, double* z_base, double* z_nms,
                     double* z_adj, double* lambda, double* evidence,
                     double* prior, char* err, int errlen) {
  return guarded(err, errlen, [&] {
    const sfi::SelectorConfig cfg = to_cfg(c);
    sfi::LogitWindow w;
    w.width = W;
    w.allowed.assign(allowed, allowed + n);
    w.values.resize(static_cast<std::size_t>(H));
    std::vector<std::vector<double>> kn(static_cast<std::size_t>(H));
    for (int h = 0; h < H; ++h) {
      w.values[h].assign(values + static_cast<std::size_t>(h) * W * n,
                         values + static_cast<std::size_t>(h + 1) * W * n);
      kn[h].assign(norms + static_cast<std::size_t>(h) * n,
                   norms + static_cast<std::size_t>(h + 1) * n);
    }
    const sfi::CacheStats stats = sfi::make_cache_stats(std::move(kn), w.allowed, cfg.epsilon);
    sfi::SelectorTrace trace;
    trace.capture_stages = true;
    const auto sel = sfi::run_selector(w, stats, cfg, &trace);
    for (int h = 0; h < H; ++h) {
      if (static_cast<int>(sel[h].size()) > out_cap)
        sfi::fail(sfi::ErrorCode::kOutOfRange, "orc_run_selector: out_cap too small");
      std::copy(sel[h].begin(), sel[h].end(), out_sel + static_cast<std::size_t>(h) * out_cap);
      out_count[h] = static_cast<int32_t>(sel[h].size());
      const std::size_t off = static_cast<std::size_t>(h) * n;
      if (z_base) std::copy(trace.stages.base[h].begin(), trace.stages.base[h].end(), z_base + off);
      if (z_nms) std::copy(trace.stages.after_nms[h].begin(), trace.stages.after_nms[h].end(), z_nms + off);
      if (z_adj) std::copy(trace.stages.after_cross[h].begin(), trace.stages.after_cross[h].end(), z_adj + off);
      if (lambda) lambda[h] = trace.fusion[h].lambda_star;
      if (evidence) std::copy(trace.fusion[h].evidence.mass.begin(), trace.fusion[h].evidence.mass.end(), evidence + off);
      if (prior) std::copy(trace.fusion[h].prior.mass.begin(), trace.fusion[h].prior.mass.end(), prior + off);
    }
  });
}

int orc_select_top_k(int n, const double* scores, const int32_t* allowed, int k,
                     int32_t* out, int32_t* out_count, char* err, int errlen) {
  return guarded(err, errlen, [&] {
    const auto sel = sfi::select_top_k(std::vector<double>(scores, scores + n),
                                       std::vector<sfi::Pos>(allowed, allowed + n), k);
    std::copy(sel.begin(), sel.end(), out);
    *out_count = static_cast<int32_t>(sel.size());
  });
}

int orc_refine_soft_nms(int n, const double* z, const orc_selector_cfg* c,
                        double* out, char* err, int errlen) {
  return guarded(err, errlen, [&] {
    const auto r = sfi::refine_soft_nms(std::vector<double>(z, z + n), to_cfg(c));
    std::copy(r.begin(), r.end(), out);
  });
}

int orc_refine_cross_head(int H, int n, const double* z, const orc_selector_cfg* c,
                          double* out, char* err, int errlen) {
  return guarded(err, errlen, [&] {
    std::vector<std::vector<double>> zz(static_cast<std::size_t>(H));
    for (int h = 0; h < H; ++h)
      zz[h].assign(z + static_cast<std::size_t>(h) * n, z + static_cast<std::size_t>(h + 1) * n);
    const auto r = sfi::refine_cross_head(zz, to_cfg(c));
    for (int h = 0; h < H; ++h)
      std::copy(r[h].begin(), r[h].end(), out + static_cast<std::size_t>(h) * n);
  });
}

void orc_recent_window(int32_t prefix_len, int n_sink, int n_recent,
                       int32_t* recent_start, int32_t* recent_len) {
  // init_decode_state + slide_recent (scheduler.cpp:60-79, 45-51)
  sfi::CacheLimits limits;
  limits.n_sink = n_sink;
  limits.n_recent = n_recent;
  limits.k_budget = 0;
  const sfi::DecodeState st = sfi::init_decode_state(prefix_len, 1, 1, limits);
  *recent_start = st.per_layer[0].recent_start;
  *recent_len = st.per_layer[0].recent_len;
}

void* orc_store_create(int n_layers, int n_kv_heads, int n_q_heads, int head_dim,
                       int max_positions, char* err, int errlen) {
  StoreBox* box = nullptr;
  const int rc = guarded(err, errlen, [&] {
    sfi::ModelSpec spec;
    spec.n_layers = n_layers;
    spec.n_kv_heads = n_kv_heads;
    spec.n_query_heads = n_q_heads;
    spec.head_dim = head_dim;
    spec.max_positions = max_positions;
    auto b = std::make_unique<StoreBox>();
    b->spec = spec;
    b->store = std::make_unique<sfi::KvStore>(spec);
    box = b.release();
  });
  return rc == 0 ? box : nullptr;
}

void orc_store_destroy(void* store) { delete static_cast<StoreBox*>(store); }

int orc_store_append(void* store, const float* k, const float* v, char* err, int errlen) {
  return guarded(err, errlen, [&] {
    StoreBox* b = static_cast<StoreBox*>(store);
    const int hd = b->spec.n_kv_heads * b->spec.head_dim;
    b->store->begin_token();
    for (int l = 0; l < b->spec.n_layers; ++l)
      b->store->append_layer(l, k + static_cast<std::size_t>(l) * hd,
                             v + static_cast<std::size_t>(l) * hd);
    b->store->end_token();
  });
}

int orc_store_append_many(void* store, int count, const float* k, const float* v,
                          char* err, int errlen) {
  return guarded(err, errlen, [&] {
    StoreBox* b = static_cast<StoreBox*>(store);
    if (b->spec.n_layers != 1)
      sfi::fail(sfi::ErrorCode::kConfig, "orc_store_append_many: one-layer stores only");
    const std::size_t hd = static_cast<std::size_t>(b->spec.n_kv_heads) * b->spec.head_dim;
    for (int i = 0; i < count; ++i) {
      b->store->begin_token();
      b->store->append_layer(0, k + i * hd, v + i * hd);
      b->store->end_token();
    }
  });
}

int32_t orc_store_size(void* store) { return static_cast<StoreBox*>(store)->store->size(); }

double orc_store_key_norm(void* store, int layer, int head, int32_t pos) {
  try {
    return static_cast<StoreBox*>(store)->store->key_norm(layer, head, pos);
  } catch (...) {
    return -1.0;
  }
}

int orc_store_reorganize(void* store, int layer, int n_sink, const int32_t* sink,
                         const int32_t* sel_counts, const int32_t* sel_flat,
                         char* err, int errlen) {
  return guarded(err, errlen, [&] {
    StoreBox* b = static_cast<StoreBox*>(store);
    b->store->reorganize(layer, std::vector<sfi::Pos>(sink, sink + n_sink),
                         unflatten(b->spec.n_kv_heads, sel_counts, sel_flat));
  });
}

int orc_store_compact(void* store, int layer, int head, int cap, int32_t* positions,
                      float* k, float* v, int32_t* count, char* err, int errlen) {
  return guarded(err, errlen, [&] {
    StoreBox* b = static_cast<StoreBox*>(store);
    const auto& seg = b->store->compact(layer, head);
    const int n = static_cast<int>(seg.positions.size());
    if (n > cap) sfi::fail(sfi::ErrorCode::kOutOfRange, "orc_store_compact: cap too small");
    std::copy(seg.positions.begin(), seg.positions.end(), positions);
    std::copy(seg.k.begin(), seg.k.end(), k);
    std::copy(seg.v.begin(), seg.v.end(), v);
    *count = n;
  });
}

int orc_attention_dense(void* store, int layer, const double* q, double* out,
                        uint64_t* reads, char* err, int errlen) {
  return guarded(err, errlen, [&] {
    StoreBox* b = static_cast<StoreBox*>(store);
    const std::size_t n = static_cast<std::size_t>(b->spec.n_query_heads) * b->spec.head_dim;
    sfi::KernelStats stats;
    const auto ctx = sfi::attention_kernel_dense(*b->store, layer, std::vector<double>(q, q + n), &stats);
    std::copy(ctx.begin(), ctx.end(), out);
    if (reads) *reads = stats.reads;
  });
}

int orc_attention_sparse(void* store, int layer, const double* q, int n_sink,
                         const int32_t* sink, const int32_t* sel_counts,
                         const int32_t* sel_flat, int32_t recent_start,
                         int32_t recent_len, double* out, uint64_t* reads,
                         char* err, int errlen) {
  return guarded(err, errlen, [&] {
    StoreBox* b = static_cast<StoreBox*>(store);
    const std::size_t n = static_cast<std::size_t>(b->spec.n_query_heads) * b->spec.head_dim;
    sfi::SupportSet support;
    support.sink.assign(sink, sink + n_sink);
    support.selected = unflatten(b->spec.n_kv_heads, sel_counts, sel_flat);
    support.recent_start = recent_start;
    support.recent_len = recent_len;
    sfi::KernelStats stats;
    const auto ctx = sfi::attention_kernel_sparse(*b->store, layer, std::vector<double>(q, q + n),
                                                  support, &stats);
    std::copy(ctx.begin(), ctx.end(), out);
    if (reads) *reads = stats.reads;
  });
}

int orc_dense_capture(void*, int, const double*, int, const int32_t*, int, double*,
                      double*, char* err, int errlen) {
  set_err(err, errlen, "capture is only reachable through the toy-model step in the reference");
  return 102;
}

/* ---- toy model + request loop (reference only) ---- */

namespace {
sfi::ModelSpec toy_spec(const orc_toy_spec* t) {
  sfi::ModelSpec spec;
  spec.n_layers = t->n_layers;
  spec.n_query_heads = t->n_query_heads;
  spec.n_kv_heads = t->n_kv_heads;
  spec.head_dim = t->head_dim;
  spec.vocab_size = t->vocab_size;
  spec.max_positions = t->max_positions;
  spec.rope_base = t->rope_base;
  return spec;
}
}  // namespace

double orc_toy_checksum(const orc_toy_spec* t, uint64_t seed) {
  try {
    const sfi::ToyModel m = sfi::ToyModel::random(toy_spec(t), seed);
    double acc = 0.0;
    auto add = [&](const Eigen::MatrixXd& w) {
      for (int r = 0; r < w.rows(); ++r)
        for (int c = 0; c < w.cols(); ++c) acc += w(r, c);
    };
    add(m.embedding());
    for (int l = 0; l < t->n_layers; ++l) {
      const auto& lw = m.layer(l);
      add(lw.wq);
      add(lw.wk);
      add(lw.wv);
      add(lw.wo);
      add(lw.w_gate);
      add(lw.w_up);
      add(lw.w_down);
    }
    add(m.lm_head());
    return acc;
  } catch (...) {
    return 0.0;
  }
}

int orc_toy_run_request(const orc_toy_spec* t, uint64_t seed, const int32_t* prompt, int plen,
                        const orc_toy_limits* lim, const orc_selector_cfg* c, int max_new,
                        int32_t* out_tokens, int32_t* out_slow, int32_t* out_cause,
                        double* out_logits, int32_t* out_sel, int32_t* out_nsel, char* err, int errlen) {
  return guarded(err, errlen, [&] {
    const sfi::ToyModel m = sfi::ToyModel::random(toy_spec(t), seed);
    sfi::CacheLimits limits;
    limits.n_sink = lim->n_sink;
    limits.n_recent = lim->n_recent;
    limits.k_budget = lim->k_budget;
    sfi::TriggerConfig trig;
    trig.trigger_tokens.assign(lim->trigger_tokens, lim->trigger_tokens + lim->n_trigger);
    trig.t_max = lim->t_max;
    trig.window_prefill = lim->window_prefill;
    sfi::RunOptions opts;
    opts.collect_logits = out_logits != nullptr;
    opts.capture_selected = out_sel != nullptr;
    const sfi::RequestResult r = sfi::run_request(m, std::vector<sfi::TokenId>(prompt, prompt + plen), limits,
                                                  trig, to_cfg(c), max_new, opts);
    for (int i = 0; i < max_new; ++i) {
      out_tokens[i] = r.tokens[i];
      out_slow[i] = r.log[i].slow ? 1 : 0;
      out_cause[i] = static_cast<int32_t>(r.log[i].cause);
      if (out_logits)
        std::copy(r.step_logits[i].begin(), r.step_logits[i].end(),
                  out_logits + static_cast<std::size_t>(i) * t->vocab_size);
      if (out_sel) {  // [max_new][n_layers][H][k_budget], counts [max_new][n_layers][H]
        const int H = t->n_kv_heads, K = lim->k_budget;
        for (int l = 0; l < t->n_layers; ++l)
          for (int h = 0; h < H; ++h) {
            const auto& v = r.selected_per_step[i][l][h];
            const std::size_t o = (static_cast<std::size_t>(i) * t->n_layers + l) * H + h;
            out_nsel[o] = static_cast<int32_t>(v.size());
            std::copy(v.begin(), v.end(), out_sel + o * K);
          }
      }
    }
  });
}

int orc_toy_run_dense(const orc_toy_spec* t, uint64_t seed, const int32_t* prompt, int plen, int max_new,
                      int32_t* out_tokens, double* out_logits, char* err, int errlen) {
  return guarded(err, errlen, [&] {
    const sfi::ToyModel m = sfi::ToyModel::random(toy_spec(t), seed);
    const sfi::DenseResult r = sfi::run_dense(m, std::vector<sfi::TokenId>(prompt, prompt + plen), max_new);
    for (int i = 0; i < max_new; ++i) {
      out_tokens[i] = r.tokens[i];
      if (out_logits)
        std::copy(r.step_logits[i].begin(), r.step_logits[i].end(),
                  out_logits + static_cast<std::size_t>(i) * t->vocab_size);
    }
  });
}

int orc_toy_capture(const orc_toy_spec* t, uint64_t seed, const int32_t* tokens, int n, int nJ,
                    const int32_t* allowed, int pool, double* out_logits, double* out_ctx, double* out_q,
                    float* out_k, float* out_v, char* err, int errlen) {
  return guarded(err, errlen, [&] {
    const sfi::ModelSpec spec = toy_spec(t);
    const sfi::ToyModel m = sfi::ToyModel::random(spec, seed);
    sfi::KvStore store(spec);
    sfi::CaptureSpec none;
    for (int i = 0; i + 1 < n; ++i) sfi::dense_attention_step(m, tokens[i], store, none);
    sfi::CaptureSpec cap;
    cap.window = true;
    cap.allowed.assign(allowed, allowed + nJ);
    cap.pool = pool == 1 ? sfi::PoolMode::kMax : sfi::PoolMode::kMean;
    cap.context = true;
    const sfi::StepOutput so = sfi::dense_attention_step(m, tokens[n - 1], store, cap);
    const int H = spec.n_kv_heads, d = spec.head_dim, hq = spec.n_query_heads;
    const sfi::LogitWindow& w = (*so.attn_logits)[0];
    for (int h = 0; h < H; ++h) std::copy(w.values[h].begin(), w.values[h].end(), out_logits + (std::size_t)h * nJ);
    std::copy(so.attn_context[0].begin(), so.attn_context[0].end(), out_ctx);
    // the layer-0 query of the last step: run_step's first lines (attention.cpp:29-33, 38-54, 342-349)
    const sfi::ToyModel::LayerWeights& lw = m.layer(0);
    const Eigen::VectorXd h0 = m.embedding().row(tokens[n - 1]).transpose();
    const double ms = h0.squaredNorm() / static_cast<double>(h0.size());
    const double inv = 1.0 / std::sqrt(ms + 1e-6);
    const Eigen::VectorXd a = (h0.array() * inv * lw.ln1.array()).matrix();
    Eigen::VectorXd q = lw.wq * a;
    const double p = static_cast<double>(store.size() - 1);
    for (int hh = 0; hh < hq; ++hh) {
      double* head = q.data() + static_cast<std::ptrdiff_t>(hh) * d;
      for (int i = 0; i < d / 2; ++i) {
        const double theta = p * std::pow(spec.rope_base, -2.0 * i / d);
        const double c = std::cos(theta), s = std::sin(theta);
        const double x = head[2 * i], y = head[2 * i + 1];
        head[2 * i] = x * c - y * s;
        head[2 * i + 1] = x * s + y * c;
      }
    }
    std::copy(q.data(), q.data() + hq * d, out_q);
    for (int pos = 1; pos <= store.size(); ++pos) {
      std::copy(store.key_at(0, pos), store.key_at(0, pos) + H * d, out_k + (std::size_t)(pos - 1) * H * d);
      std::copy(store.value_at(0, pos), store.value_at(0, pos) + H * d, out_v + (std::size_t)(pos - 1) * H * d);
    }
  });
}

}  // extern "C"

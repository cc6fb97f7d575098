/*
 * sfi_oracle.c — CPU ORACLE (test infrastructure only; never on the product
 * path). A line-faithful plain-C restatement ("port") of the reference's SFI
 * hot path, implementing oracle/oracle_abi.h. Each function cites the
 * reference file:line it restates (paths relative to /root/reference/proj).
 *
 * Pinning: tests/test_oracle.py checks this port bit-for-bit against the
 * unmodified reference (oracle/_ref/libsfi_ref.so, built from the reference
 * sources) on seeded inputs, and against the reference's known-answer tests
 * (tests/golden/). Arithmetic is fp64 with the reference's sequential
 * summation orders; compiled without FMA contraction (-ffp-contract=off) and
 * against the same glibc libm, so results are bit-identical.
 */
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "oracle_abi.h"

/* sfi::ErrorCode + 1 (error.hpp:23-34) */
enum {
  E_CONFIG = 1,
  E_EMPTY_SUPPORT = 2,
  E_SUPPORT_MISMATCH = 3,
  E_NON_FINITE = 4,
  E_OVERLAP = 5,
  E_STALE_COMPACT = 6,
  E_OUT_OF_RANGE = 7,
  E_CONTEXT_OVERFLOW = 9,
  E_ALLOC = 200
};

static const double kMaskedLogit = -1e30; /* selector.hpp:42 */

static int fail(char* err, int errlen, int code, const char* fmt, ...) {
  if (err && errlen > 0) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(err, (size_t)errlen, fmt, ap);
    va_end(ap);
  }
  return code;
}

/* std::max / std::min / std::clamp semantics (libstdc++) */
static double dmax(double a, double b) { return (a < b) ? b : a; }
static double dclamp(double v, double lo, double hi) {
  return (v < lo) ? lo : (hi < v) ? hi : v;
}

const char* orc_kind(void) { return "port"; }

/* ------------------------------------------------------------------------ */
/* distribution.cpp                                                          */

/* normalize (distribution.cpp:41-60): sequential sum, then w / sum. */
static int normalize_inplace(int n, double* w, char* err, int errlen) {
  if (n == 0) return fail(err, errlen, E_EMPTY_SUPPORT, "normalize: empty support");
  double sum = 0.0;
  for (int i = 0; i < n; ++i) {
    if (!isfinite(w[i]) || w[i] < 0.0)
      return fail(err, errlen, E_NON_FINITE, "normalize: weights must be finite and >= 0");
    sum += w[i];
  }
  if (sum <= 0.0) return fail(err, errlen, E_EMPTY_SUPPORT, "normalize: all weights are zero");
  for (int i = 0; i < n; ++i) w[i] = w[i] / sum;
  return 0;
}

/* dot / squared_norm (distribution.cpp:66-78) */
static double dot(int n, const double* a, const double* b) {
  double acc = 0.0;
  for (int i = 0; i < n; ++i) acc += a[i] * b[i];
  return acc;
}
static double squared_norm(int n, const double* a) {
  double acc = 0.0;
  for (int i = 0; i < n; ++i) acc += a[i] * a[i];
  return acc;
}

/* ------------------------------------------------------------------------ */
/* selector.cpp                                                              */

/* evidence_from_window (selector.cpp:96-127) with row_softmax (:54-74) for
 * one head. values: [W*n]; f: [n] out; scratch p: [n]. */
static int evidence_head(int W, int n, const double* values, double alpha,
                         double* f, double* p, char* err, int errlen) {
  for (int j = 0; j < n; ++j) f[j] = 0.0; /* mu */
  for (int row = 0; row < W; ++row) {
    const double* v = values + (size_t)row * n;
    double max_logit = kMaskedLogit;
    for (int j = 0; j < n; ++j) {
      if (!isfinite(v[j]))
        return fail(err, errlen, E_NON_FINITE, "evidence_from_window: non-finite logit");
      max_logit = dmax(max_logit, v[j]);
    }
    double sum = 0.0;
    for (int j = 0; j < n; ++j) {
      p[j] = (v[j] <= kMaskedLogit) ? 0.0 : exp(v[j] - max_logit);
      sum += p[j];
    }
    if (sum <= 0.0)
      return fail(err, errlen, E_EMPTY_SUPPORT, "evidence_from_window: fully masked row");
    for (int j = 0; j < n; ++j) p[j] /= sum;
    for (int j = 0; j < n; ++j) f[j] += pow(p[j], alpha);
  }
  const double inv_w = 1.0 / (double)W;
  for (int j = 0; j < n; ++j) f[j] = pow(f[j] * inv_w, 1.0 / alpha);
  return normalize_inplace(n, f, err, errlen);
}

/* prior_from_stats (selector.cpp:129-160) for one head; u from
 * make_cache_stats (:78-94). */
static int prior_head(int n, const double* norms, const double* u,
                      const orc_selector_cfg* cfg, double* r, char* err, int errlen) {
  for (int j = 0; j < n; ++j) {
    const double norm = norms[j];
    if (!isfinite(norm) || norm < 0.0)
      return fail(err, errlen, E_NON_FINITE, "prior_from_stats: bad key norm");
    const double pi_kn = pow(norm + cfg->epsilon, -cfg->gamma);
    const double pi_pos =
        exp(-cfg->beta * pow(u[j], cfg->p_curve)) * pow(1.0 - u[j] + cfg->epsilon, cfg->eta);
    r[j] = pi_kn * pi_pos;
  }
  return normalize_inplace(n, r, err, errlen);
}

/* fuse (selector.cpp:162-185) -> s, lambda */
static double fuse_head(int n, const double* f, const double* r,
                        const orc_selector_cfg* cfg, double* s) {
  const double ff = squared_norm(n, f);
  const double fr = dot(n, f, r);
  const double rr = squared_norm(n, r);
  const double denom = ff - 2.0 * fr + rr;
  double lambda = 0.0;
  if (fabs(denom) >= cfg->epsilon) {
    lambda = (ff - fr) / denom;
    lambda = dclamp(lambda, 0.0, cfg->lambda_clip);
  }
  for (int j = 0; j < n; ++j) s[j] = (1.0 - lambda) * f[j] + lambda * r[j];
  return lambda;
}

/* refine_soft_nms (selector.cpp:187-202) */
static void soft_nms(int n, const double* z, const orc_selector_cfg* cfg, double* out) {
  for (int j = 0; j < n; ++j) {
    const int lo = (j - cfg->nms_radius > 0) ? j - cfg->nms_radius : 0;
    const int hi = (j + cfg->nms_radius < n - 1) ? j + cfg->nms_radius : n - 1;
    double m = z[j];
    for (int i = lo; i <= hi; ++i) m = dmax(m, z[i]);
    const double gap = m - z[j];
    out[j] = z[j] - cfg->alpha_soft * gap;
  }
}

/* refine_cross_head (selector.cpp:204-230); z, out: [H][n] */
static int cross_head(int H, int n, const double* z, const orc_selector_cfg* cfg,
                      double* out, char* err, int errlen) {
  if (H == 0) return 0;
  double* resp = (double*)malloc(sizeof(double) * (size_t)H);
  if (!resp) return fail(err, errlen, E_ALLOC, "cross_head: out of memory");
  for (int j = 0; j < n; ++j) {
    double max_s = z[j];
    for (int h = 1; h < H; ++h) max_s = dmax(max_s, z[(size_t)h * n + j]);
    double sum = 0.0;
    for (int h = 0; h < H; ++h) {
      resp[h] = exp((z[(size_t)h * n + j] - max_s) / cfg->temperature);
      sum += resp[h];
    }
    for (int h = 0; h < H; ++h) {
      const double r = resp[h] / sum;
      out[(size_t)h * n + j] =
          z[(size_t)h * n + j] + cfg->alpha_cross * log(dmax(r, cfg->epsilon));
    }
  }
  free(resp);
  return 0;
}

/* select_top_k (selector.cpp:232-252): (score desc, position asc) total
 * order, picked positions returned ascending. */
static const double* g_scores;
static const int32_t* g_allowed;
static int cmp_rank(const void* a, const void* b) {
  const int ia = *(const int*)a, ib = *(const int*)b;
  if (g_scores[ia] != g_scores[ib]) return g_scores[ia] > g_scores[ib] ? -1 : 1;
  return (g_allowed[ia] < g_allowed[ib]) ? -1 : (g_allowed[ia] > g_allowed[ib]) ? 1 : 0;
}
static int cmp_pos(const void* a, const void* b) {
  const int32_t pa = *(const int32_t*)a, pb = *(const int32_t*)b;
  return (pa < pb) ? -1 : (pa > pb) ? 1 : 0;
}

int orc_select_top_k(int n, const double* scores, const int32_t* allowed, int k,
                     int32_t* out, int32_t* out_count, char* err, int errlen) {
  if (k < 0) return fail(err, errlen, E_OUT_OF_RANGE, "select_top_k: negative budget");
  *out_count = 0;
  if (k == 0) return 0;
  if (n <= k) {
    memcpy(out, allowed, sizeof(int32_t) * (size_t)n);
    *out_count = n;
    return 0;
  }
  int* order = (int*)malloc(sizeof(int) * (size_t)n);
  if (!order) return fail(err, errlen, E_ALLOC, "select_top_k: out of memory");
  for (int i = 0; i < n; ++i) order[i] = i;
  g_scores = scores;
  g_allowed = allowed;
  qsort(order, (size_t)n, sizeof(int), cmp_rank);
  for (int i = 0; i < k; ++i) out[i] = allowed[order[i]];
  qsort(out, (size_t)k, sizeof(int32_t), cmp_pos);
  *out_count = k;
  free(order);
  return 0;
}

int orc_refine_soft_nms(int n, const double* z, const orc_selector_cfg* cfg,
                        double* out, char* err, int errlen) {
  (void)err;
  (void)errlen;
  soft_nms(n, z, cfg, out);
  return 0;
}

int orc_refine_cross_head(int H, int n, const double* z, const orc_selector_cfg* cfg,
                          double* out, char* err, int errlen) {
  return cross_head(H, n, z, cfg, out, err, errlen);
}

/* run_selector (selector.cpp:254-299) */
int orc_run_selector(int H, int W, int n, const int32_t* allowed,
                     const double* values, const double* norms,
                     const orc_selector_cfg* cfg, int32_t* out_sel, int out_cap,
                     int32_t* out_count, double* z_base_out, double* z_nms_out,
                     double* z_adj_out, double* lambda_out, double* evidence_out,
                     double* prior_out, char* err, int errlen) {
  if (n == 0) return fail(err, errlen, E_EMPTY_SUPPORT, "make_cache_stats: empty allowed set");
  if (W < 1) return fail(err, errlen, E_OUT_OF_RANGE, "evidence_from_window: window width must be >= 1");
  const size_t hn = (size_t)H * n;
  double* f = (double*)malloc(sizeof(double) * hn);
  double* r = (double*)malloc(sizeof(double) * hn);
  double* zb = (double*)malloc(sizeof(double) * hn);
  double* zn = (double*)malloc(sizeof(double) * hn);
  double* za = (double*)malloc(sizeof(double) * hn);
  double* p = (double*)malloc(sizeof(double) * (size_t)n);
  double* u = (double*)malloc(sizeof(double) * (size_t)n);
  int rc = 0;
  if (!f || !r || !zb || !zn || !za || !p || !u) {
    rc = fail(err, errlen, E_ALLOC, "run_selector: out of memory");
    goto done;
  }
  /* make_cache_stats (selector.cpp:87-92) */
  {
    const int32_t j_min = allowed[0], j_max = allowed[n - 1];
    const double denom = (double)(j_max - j_min) + cfg->epsilon;
    for (int i = 0; i < n; ++i) u[i] = (double)(allowed[i] - j_min) / denom;
  }
  /* Stage A: evidence for every head, then prior for every head
   * (selector.cpp:262-264) */
  for (int h = 0; h < H; ++h) {
    rc = evidence_head(W, n, values + (size_t)h * W * n, cfg->alpha, f + (size_t)h * n, p, err, errlen);
    if (rc) goto done;
  }
  for (int h = 0; h < H; ++h) {
    rc = prior_head(n, norms + (size_t)h * n, u, cfg, r + (size_t)h * n, err, errlen);
    if (rc) goto done;
  }
  for (int h = 0; h < H; ++h) {
    double* s = p; /* scratch */
    const double lam = fuse_head(n, f + (size_t)h * n, r + (size_t)h * n, cfg, s);
    if (lambda_out) lambda_out[h] = lam;
    for (int j = 0; j < n; ++j) zb[(size_t)h * n + j] = log(s[j] + cfg->epsilon);
  }
  /* Stage B (selector.cpp:279-297) */
  for (int h = 0; h < H; ++h) soft_nms(n, zb + (size_t)h * n, cfg, zn + (size_t)h * n);
  rc = cross_head(H, n, zn, cfg, za, err, errlen);
  if (rc) goto done;
  for (int h = 0; h < H; ++h) {
    const int expect = (cfg->k_budget < n) ? cfg->k_budget : n;
    if (expect > out_cap) {
      rc = fail(err, errlen, E_OUT_OF_RANGE, "orc_run_selector: out_cap too small");
      goto done;
    }
    rc = orc_select_top_k(n, za + (size_t)h * n, allowed, cfg->k_budget,
                          out_sel + (size_t)h * out_cap, out_count + h, err, errlen);
    if (rc) goto done;
  }
  if (z_base_out) memcpy(z_base_out, zb, sizeof(double) * hn);
  if (z_nms_out) memcpy(z_nms_out, zn, sizeof(double) * hn);
  if (z_adj_out) memcpy(z_adj_out, za, sizeof(double) * hn);
  if (evidence_out) memcpy(evidence_out, f, sizeof(double) * hn);
  if (prior_out) memcpy(prior_out, r, sizeof(double) * hn);
done:
  free(f);
  free(r);
  free(zb);
  free(zn);
  free(za);
  free(p);
  free(u);
  return rc;
}

/* ------------------------------------------------------------------------ */
/* scheduler.cpp                                                             */

/* init_decode_state + slide_recent (scheduler.cpp:60-79, 45-51) */
void orc_recent_window(int32_t prefix_len, int n_sink, int n_recent,
                       int32_t* recent_start, int32_t* recent_len) {
  const int sink = (n_sink < prefix_len) ? n_sink : prefix_len;
  int len = prefix_len - sink;
  if (len < 0) len = 0;
  if (len > n_recent) len = n_recent;
  *recent_len = len;
  *recent_start = prefix_len - len + 1;
}

/* ------------------------------------------------------------------------ */
/* attention.cpp: KvStore                                                    */

typedef struct {
  int32_t* positions;
  float* k;
  float* v;
  int count;
} Compact;

typedef struct {
  float* k_paged; /* [cap][H][d] */
  float* v_paged;
  double* norms; /* [H][cap] */
  Compact* compact; /* [H] */
  int compact_valid;
} Layer;

typedef struct {
  int n_layers, H, Hq, d, max_positions;
  int32_t len, cap;
  Layer* layers;
} Store;

void* orc_store_create(int n_layers, int n_kv_heads, int n_q_heads, int head_dim,
                       int max_positions, char* err, int errlen) {
  /* ModelSpec::validate (model.cpp:113-123), the parts KvStore relies on */
  if (n_layers < 1 || n_kv_heads < 1 || n_q_heads < 1 || n_q_heads % n_kv_heads != 0 ||
      head_dim < 2 || head_dim % 2 != 0 || max_positions < 1) {
    fail(err, errlen, E_CONFIG, "model spec: invalid shape");
    return NULL;
  }
  Store* s = (Store*)calloc(1, sizeof(Store));
  s->n_layers = n_layers;
  s->H = n_kv_heads;
  s->Hq = n_q_heads;
  s->d = head_dim;
  s->max_positions = max_positions;
  s->layers = (Layer*)calloc((size_t)n_layers, sizeof(Layer));
  for (int l = 0; l < n_layers; ++l)
    s->layers[l].compact = (Compact*)calloc((size_t)n_kv_heads, sizeof(Compact));
  return s;
}

void orc_store_destroy(void* store) {
  Store* s = (Store*)store;
  if (!s) return;
  for (int l = 0; l < s->n_layers; ++l) {
    Layer* L = &s->layers[l];
    free(L->k_paged);
    free(L->v_paged);
    free(L->norms);
    for (int h = 0; h < s->H; ++h) {
      free(L->compact[h].positions);
      free(L->compact[h].k);
      free(L->compact[h].v);
    }
    free(L->compact);
  }
  free(s->layers);
  free(s);
}

static int grow(Store* s, int32_t need) {
  if (need <= s->cap) return 0;
  int32_t cap = s->cap ? s->cap : 64;
  while (cap < need) cap *= 2;
  const size_t hd = (size_t)s->H * s->d;
  for (int l = 0; l < s->n_layers; ++l) {
    Layer* L = &s->layers[l];
    float* k = (float*)realloc(L->k_paged, sizeof(float) * hd * (size_t)cap);
    float* v = (float*)realloc(L->v_paged, sizeof(float) * hd * (size_t)cap);
    double* nm = (double*)malloc(sizeof(double) * (size_t)s->H * (size_t)cap);
    if (!k || !v || !nm) return 1;
    for (int h = 0; h < s->H; ++h)
      if (s->len) memcpy(nm + (size_t)h * cap, L->norms + (size_t)h * s->cap, sizeof(double) * (size_t)s->len);
    free(L->norms);
    L->k_paged = k;
    L->v_paged = v;
    L->norms = nm;
  }
  s->cap = cap;
  return 0;
}

/* begin_token / append_layer / end_token (attention.cpp:128-159); the key
 * norm is sqrt of the sequential fp64 sum of squares (:143-150). */
static int append_one(Store* s, int layer, const float* k, const float* v) {
  const size_t hd = (size_t)s->H * s->d;
  Layer* L = &s->layers[layer];
  memcpy(L->k_paged + (size_t)s->len * hd, k, sizeof(float) * hd);
  memcpy(L->v_paged + (size_t)s->len * hd, v, sizeof(float) * hd);
  for (int h = 0; h < s->H; ++h) {
    double acc = 0.0;
    for (int c = 0; c < s->d; ++c) {
      const double x = (double)k[h * s->d + c];
      acc += x * x;
    }
    L->norms[(size_t)h * s->cap + s->len] = sqrt(acc);
  }
  return 0;
}

int orc_store_append(void* store, const float* k, const float* v, char* err, int errlen) {
  Store* s = (Store*)store;
  if (s->len >= s->max_positions)
    return fail(err, errlen, E_CONTEXT_OVERFLOW, "KvStore: max_positions exceeded");
  if (grow(s, s->len + 1)) return fail(err, errlen, E_ALLOC, "KvStore: out of memory");
  const size_t hd = (size_t)s->H * s->d;
  for (int l = 0; l < s->n_layers; ++l) append_one(s, l, k + l * hd, v + l * hd);
  s->len += 1;
  return 0;
}

int orc_store_append_many(void* store, int count, const float* k, const float* v,
                          char* err, int errlen) {
  Store* s = (Store*)store;
  if (s->n_layers != 1) return fail(err, errlen, E_CONFIG, "orc_store_append_many: one-layer stores only");
  if (s->len + count > s->max_positions)
    return fail(err, errlen, E_CONTEXT_OVERFLOW, "KvStore: max_positions exceeded");
  if (grow(s, s->len + count)) return fail(err, errlen, E_ALLOC, "KvStore: out of memory");
  const size_t hd = (size_t)s->H * s->d;
  for (int i = 0; i < count; ++i) {
    append_one(s, 0, k + i * hd, v + i * hd);
    s->len += 1;
  }
  return 0;
}

int32_t orc_store_size(void* store) { return ((Store*)store)->len; }

double orc_store_key_norm(void* store, int layer, int head, int32_t pos) {
  Store* s = (Store*)store;
  if (pos < 1 || pos > s->len) return -1.0;
  return s->layers[layer].norms[(size_t)head * s->cap + (pos - 1)];
}

/* KvStore::reorganize (attention.cpp:186-217): per head merge(sink,
 * selected) ascending, strictly-increasing check, range check, then a pure
 * fp32 row copy from paged storage. */
int orc_store_reorganize(void* store, int layer, int n_sink, const int32_t* sink,
                         const int32_t* sel_counts, const int32_t* sel_flat,
                         char* err, int errlen) {
  Store* s = (Store*)store;
  Layer* L = &s->layers[layer];
  const int d = s->d;
  const size_t hd = (size_t)s->H * d;
  size_t off = 0;
  for (int h = 0; h < s->H; ++h) {
    const int ns = sel_counts[h];
    const int32_t* sel = sel_flat + off;
    off += (size_t)ns;
    const int m = n_sink + ns;
    int32_t* merged = (int32_t*)malloc(sizeof(int32_t) * (size_t)(m ? m : 1));
    /* std::merge: on equal keys the first range's element comes first */
    int a = 0, b = 0, o = 0;
    while (a < n_sink && b < ns) merged[o++] = (sel[b] < sink[a]) ? sel[b++] : sink[a++];
    while (a < n_sink) merged[o++] = sink[a++];
    while (b < ns) merged[o++] = sel[b++];
    for (int i = 0; i + 1 < m; ++i)
      if (merged[i] >= merged[i + 1]) {
        free(merged);
        return fail(err, errlen, E_OVERLAP, "reorganize: sink and selected sets overlap or are unsorted");
      }
    Compact* c = &L->compact[h];
    free(c->positions);
    free(c->k);
    free(c->v);
    c->positions = merged;
    c->count = m;
    c->k = (float*)malloc(sizeof(float) * (size_t)(m ? m : 1) * d);
    c->v = (float*)malloc(sizeof(float) * (size_t)(m ? m : 1) * d);
    for (int i = 0; i < m; ++i) {
      const int32_t pos = merged[i];
      if (pos < 1 || pos > s->len)
        return fail(err, errlen, E_OUT_OF_RANGE, "reorganize: position %d not written", pos);
      const size_t src = (size_t)(pos - 1) * hd + (size_t)h * d;
      memcpy(c->k + (size_t)i * d, L->k_paged + src, sizeof(float) * d);
      memcpy(c->v + (size_t)i * d, L->v_paged + src, sizeof(float) * d);
    }
  }
  L->compact_valid = 1;
  return 0;
}

int orc_store_compact(void* store, int layer, int head, int cap, int32_t* positions,
                      float* k, float* v, int32_t* count, char* err, int errlen) {
  Store* s = (Store*)store;
  const Compact* c = &s->layers[layer].compact[head];
  if (c->count > cap) return fail(err, errlen, E_OUT_OF_RANGE, "orc_store_compact: cap too small");
  if (c->count) {
    memcpy(positions, c->positions, sizeof(int32_t) * (size_t)c->count);
    memcpy(k, c->k, sizeof(float) * (size_t)c->count * s->d);
    memcpy(v, c->v, sizeof(float) * (size_t)c->count * s->d);
  }
  *count = c->count;
  return 0;
}

/* compact_matches (attention.cpp:219-231) */
static int compact_matches(Store* s, int layer, int n_sink, const int32_t* sink,
                           const int32_t* sel_counts, const int32_t* sel_flat) {
  Layer* L = &s->layers[layer];
  if (!L->compact_valid) return 0;
  size_t off = 0;
  for (int h = 0; h < s->H; ++h) {
    const int ns = sel_counts[h];
    const int32_t* sel = sel_flat + off;
    off += (size_t)ns;
    const Compact* c = &L->compact[h];
    if (c->count != n_sink + ns) return 0;
    int a = 0, b = 0, o = 0;
    while (a < n_sink || b < ns) {
      int32_t nxt;
      if (a < n_sink && (b >= ns || !(sel[b] < sink[a])))
        nxt = sink[a++];
      else
        nxt = sel[b++];
      if (c->positions[o++] != nxt) return 0;
    }
  }
  return 1;
}

typedef struct {
  const float* k;
  const float* v;
  int count;
  int stride;
} Seg;

/* attend (attention.cpp:80-113): two-pass fp64 softmax over the segments.
 * logits (entry order) are returned in `logits`. */
static void attend(const double* q, const Seg* segs, int n_segs, int total, int d,
                   double inv_sqrt_d, double* logits, double* out) {
  double max_logit = -INFINITY;
  int idx = 0;
  for (int s = 0; s < n_segs; ++s)
    for (int i = 0; i < segs[s].count; ++i) {
      const float* kp = segs[s].k + (size_t)i * segs[s].stride;
      double acc = 0.0;
      for (int c = 0; c < d; ++c) acc += q[c] * (double)kp[c];
      const double logit = acc * inv_sqrt_d;
      logits[idx++] = logit;
      max_logit = dmax(max_logit, logit);
    }
  (void)total;
  double exp_sum = 0.0;
  for (int c = 0; c < d; ++c) out[c] = 0.0;
  idx = 0;
  for (int s = 0; s < n_segs; ++s)
    for (int i = 0; i < segs[s].count; ++i) {
      const double w = exp(logits[idx++] - max_logit);
      exp_sum += w;
      const float* vp = segs[s].v + (size_t)i * segs[s].stride;
      for (int c = 0; c < d; ++c) out[c] += w * (double)vp[c];
    }
  const double inv = 1.0 / exp_sum;
  for (int c = 0; c < d; ++c) out[c] *= inv;
}

/* attention_kernel_dense (attention.cpp:502-523) plus the slow-step capture
 * of run_step (attention.cpp:367-375, 394-409): W = 1, positions j > size()
 * are masked (never in decode). */
static int dense_impl(Store* s, int layer, const double* q, double* out, uint64_t* reads,
                      int nJ, const int32_t* allowed, int pool, double* logits_out,
                      char* err, int errlen) {
  if (s->len < 1) return fail(err, errlen, E_OUT_OF_RANGE, "KvStore: position 1 not written");
  const int d = s->d, H = s->H, group = s->Hq / s->H;
  const double inv_sqrt_d = 1.0 / sqrt((double)d);
  Layer* L = &s->layers[layer];
  double* scratch = (double*)malloc(sizeof(double) * (size_t)s->len);
  if (!scratch) return fail(err, errlen, E_ALLOC, "dense: out of memory");
  if (reads) *reads = 0;
  for (int head = 0; head < H; ++head) {
    Seg seg = {L->k_paged + (size_t)head * d, L->v_paged + (size_t)head * d, s->len, H * d};
    if (reads) *reads += (uint64_t)s->len;
    double* row = logits_out ? logits_out + (size_t)head * nJ : NULL;
    if (row)
      for (int c = 0; c < nJ; ++c) row[c] = (pool == 1) ? kMaskedLogit : 0.0;
    for (int g = 0; g < group; ++g) {
      const int qh = head * group + g;
      attend(q + (size_t)qh * d, &seg, 1, s->len, d, inv_sqrt_d, scratch, out + (size_t)qh * d);
      if (row) {
        for (int c = 0; c < nJ; ++c) {
          const int32_t j = allowed[c];
          if (j > s->len) {
            row[c] = kMaskedLogit;
            continue;
          }
          const double logit = scratch[j - 1];
          if (pool == 0)
            row[c] += logit / group;
          else
            row[c] = dmax(row[c], logit);
        }
      }
    }
  }
  free(scratch);
  return 0;
}

int orc_attention_dense(void* store, int layer, const double* q, double* out,
                        uint64_t* reads, char* err, int errlen) {
  return dense_impl((Store*)store, layer, q, out, reads, 0, NULL, 0, NULL, err, errlen);
}

int orc_dense_capture(void* store, int layer, const double* q, int nJ,
                      const int32_t* allowed, int pool, double* out, double* logits,
                      char* err, int errlen) {
  Store* s = (Store*)store;
  for (int c = 0; c < nJ; ++c)
    if (allowed[c] < 1 || allowed[c] > s->len)
      return fail(err, errlen, E_OUT_OF_RANGE, "dense_attention_step: allowed position %d out of range",
                  allowed[c]);
  return dense_impl(s, layer, q, out, NULL, nJ, allowed, pool, logits, err, errlen);
}

/* attention_kernel_sparse (attention.cpp:525-550) with sparse_segments
 * (:270-291): compact (stride d) first, then the paged recent tail. */
int orc_attention_sparse(void* store, int layer, const double* q, int n_sink,
                         const int32_t* sink, const int32_t* sel_counts,
                         const int32_t* sel_flat, int32_t recent_start,
                         int32_t recent_len, double* out, uint64_t* reads,
                         char* err, int errlen) {
  Store* s = (Store*)store;
  if (!compact_matches(s, layer, n_sink, sink, sel_counts, sel_flat))
    return fail(err, errlen, E_STALE_COMPACT,
                "attention_kernel_sparse: compact buffer does not match the support");
  const int d = s->d, H = s->H, group = s->Hq / s->H;
  const double inv_sqrt_d = 1.0 / sqrt((double)d);
  Layer* L = &s->layers[layer];
  if (recent_len > 0 && (recent_start < 1 || recent_start + recent_len - 1 > s->len))
    return fail(err, errlen, E_OUT_OF_RANGE, "KvStore: position %d not written", recent_start);
  int max_total = recent_len;
  for (int h = 0; h < H; ++h)
    if (L->compact[h].count + recent_len > max_total) max_total = L->compact[h].count + recent_len;
  double* scratch = (double*)malloc(sizeof(double) * (size_t)(max_total ? max_total : 1));
  if (reads) *reads = 0;
  for (int head = 0; head < H; ++head) {
    Seg segs[2];
    int n = 0, total = 0;
    const Compact* c = &L->compact[head];
    if (c->count > 0) {
      segs[n].k = c->k;
      segs[n].v = c->v;
      segs[n].count = c->count;
      segs[n].stride = d;
      total += c->count;
      ++n;
    }
    if (recent_len > 0) {
      const size_t off = (size_t)(recent_start - 1) * H * d + (size_t)head * d;
      segs[n].k = L->k_paged + off;
      segs[n].v = L->v_paged + off;
      segs[n].count = recent_len;
      segs[n].stride = H * d;
      total += recent_len;
      ++n;
    }
    if (total == 0) {
      free(scratch);
      return fail(err, errlen, E_EMPTY_SUPPORT, "sparse_attention_step: empty support");
    }
    if (reads) *reads += (uint64_t)total;
    for (int g = 0; g < group; ++g) {
      const int qh = head * group + g;
      attend(q + (size_t)qh * d, segs, n, total, d, inv_sqrt_d, scratch, out + (size_t)qh * d);
    }
  }
  free(scratch);
  return 0;
}

/*
 * oracle_abi.h — C ABI of the CPU ORACLE (test infrastructure only).
 *
 * Two libraries implement this header with identical semantics:
 *   oracle/_ref/libsfi_ref.so  — the UNMODIFIED reference sources from
 *       /root/reference/proj/src/{selector,distribution,config,attention,
 *       model,scheduler,oracle}.cpp compiled by oracle/Makefile against the
 *       Eigen-API shim, wrapped by oracle/ref_capi.cpp;
 *   oracle/liboracle.so         — oracle/sfi_oracle.c, a line-faithful plain-C
 *       restatement ("port") of the same reference functions.
 * Only tests/, __graft_entry__.smoke() and bench.py's CPU arms may load
 * either library, and only as the checker / CPU baseline. The product path
 * (paper_2603_12038_b200) never links or calls anything here.
 *
 * Conventions follow the reference: positions are 1-based int32
 * (distribution.hpp:23-26); KV storage is fp32 [len][H][d] per layer
 * (attention.cpp:141-142); attention math is fp64. Status codes are 0 on
 * success, else 1 + sfi::ErrorCode (error.hpp:23-34); the message is copied
 * into err[errlen].
 */
#ifndef SFI_ORACLE_ABI_H
#define SFI_ORACLE_ABI_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif
#pragma GCC visibility push(default)

typedef struct {
  double alpha, gamma, beta, p_curve, eta, lambda_clip, alpha_soft, alpha_cross,
      temperature, epsilon;
  int32_t nms_radius, k_budget, pool; /* pool: 0 = mean, 1 = max */
} orc_selector_cfg;

/* Which implementation this is: "reference" or "port". */
const char* orc_kind(void);

/* run_selector (selector.cpp:254-299) on a W x |J| window per head.
 * values: [H][W*n]; allowed: [n] ascending; norms: [H][n] (the CacheStats
 * key norms, built with make_cache_stats selector.cpp:78-94).
 * out_sel: [H][out_cap] ascending positions, out_count: [H].
 * Optional stage dumps (NULL to skip): z_base/z_nms/z_adj [H][n], lambda [H],
 * evidence/prior [H][n]. */
int orc_run_selector(int H, int W, int n, const int32_t* allowed,
                     const double* values, const double* norms,
                     const orc_selector_cfg* cfg, int32_t* out_sel, int out_cap,
                     int32_t* out_count, double* z_base, double* z_nms,
                     double* z_adj, double* lambda, double* evidence,
                     double* prior, char* err, int errlen);

/* select_top_k (selector.cpp:232-252). out: [max(0,min(k,n))]. */
int orc_select_top_k(int n, const double* scores, const int32_t* allowed, int k,
                     int32_t* out, int32_t* out_count, char* err, int errlen);

/* Individual Selector stages (selector.hpp:88-122), one head at a time. */
int orc_refine_soft_nms(int n, const double* z, const orc_selector_cfg* cfg,
                        double* out, char* err, int errlen);
int orc_refine_cross_head(int H, int n, const double* z,
                          const orc_selector_cfg* cfg, double* out, char* err,
                          int errlen);

/* Scheduler semantics (scheduler.cpp:45-51, 81-99). */
void orc_recent_window(int32_t prefix_len, int n_sink, int n_recent,
                       int32_t* recent_start, int32_t* recent_len);

/* ---- KV store (attention.hpp:100-155) ---- */
void* orc_store_create(int n_layers, int n_kv_heads, int n_q_heads, int head_dim,
                       int max_positions, char* err, int errlen);
void orc_store_destroy(void* store);
/* Appends one token for every layer (begin_token / append_layer / end_token):
 * k, v: [n_layers][H*d] fp32. */
int orc_store_append(void* store, const float* k, const float* v, char* err,
                     int errlen);
/* Appends `count` tokens for ONE-layer stores from [count][H*d] arrays. */
int orc_store_append_many(void* store, int count, const float* k,
                          const float* v, char* err, int errlen);
int32_t orc_store_size(void* store);
double orc_store_key_norm(void* store, int layer, int head, int32_t pos);
/* KvStore::reorganize: sink [n_sink]; selected flattened per head with
 * counts sel_counts[H]. */
int orc_store_reorganize(void* store, int layer, int n_sink, const int32_t* sink,
                         const int32_t* sel_counts, const int32_t* sel_flat,
                         char* err, int errlen);
/* Copies compact(layer, head): positions [cap], k/v [cap*d]. */
int orc_store_compact(void* store, int layer, int head, int cap,
                      int32_t* positions, float* k, float* v, int32_t* count,
                      char* err, int errlen);
/* attention_kernel_dense (attention.cpp:502-523): q [Hq*d] -> out [Hq*d].
 * reads = stats.reads. */
int orc_attention_dense(void* store, int layer, const double* q, double* out,
                        uint64_t* reads, char* err, int errlen);
/* attention_kernel_sparse (attention.cpp:525-550). */
int orc_attention_sparse(void* store, int layer, const double* q, int n_sink,
                         const int32_t* sink, const int32_t* sel_counts,
                         const int32_t* sel_flat, int32_t recent_start,
                         int32_t recent_len, double* out, uint64_t* reads,
                         char* err, int errlen);
/* Slow-step pooled-logit capture over J (attention.cpp:367-409 at W=1):
 * dense attention over positions 1..size() for every q head, plus per KV
 * head the pooled (mean: row += logit/G from 0.0; max: from kMaskedLogit)
 * raw logits over allowed[nJ]. logits: [H][nJ]. Port only (the reference
 * exposes capture solely through the toy-model step). */
int orc_dense_capture(void* store, int layer, const double* q, int nJ,
                      const int32_t* allowed, int pool, double* out,
                      double* logits, char* err, int errlen);

/* ---- Toy model + request loop: REFERENCE LIBRARY ONLY (the port does not
 * restate the toy decoder). ToyModel::random (model.cpp:141-167),
 * run_request (scheduler.cpp:213-330), run_dense (:332-365). ---- */
typedef struct {
  int32_t n_layers, n_query_heads, n_kv_heads, head_dim, vocab_size, max_positions;
  double rope_base;
} orc_toy_spec;
typedef struct {
  int32_t n_sink, n_recent, k_budget; /* CacheLimits */
  const int32_t* trigger_tokens;      /* TriggerConfig */
  int32_t n_trigger, t_max, window_prefill;
} orc_toy_limits;
/* Order-fixed sum of every weight of ToyModel::random(spec, seed). */
double orc_toy_checksum(const orc_toy_spec* spec, uint64_t seed);
/* out_tokens / out_slow / out_cause (StepCause) [max_new]; out_logits
 * [max_new][vocab] or NULL; out_sel [max_new][n_layers][H][k_budget] with
 * out_nsel [max_new][n_layers][H] (the selected sets after each step) or NULL. */
int orc_toy_run_request(const orc_toy_spec* spec, uint64_t seed, const int32_t* prompt, int plen,
                        const orc_toy_limits* limits, const orc_selector_cfg* cfg, int max_new,
                        int32_t* out_tokens, int32_t* out_slow, int32_t* out_cause,
                        double* out_logits, int32_t* out_sel, int32_t* out_nsel, char* err, int errlen);
int orc_toy_run_dense(const orc_toy_spec* spec, uint64_t seed, const int32_t* prompt, int plen,
                      int max_new, int32_t* out_tokens, double* out_logits, char* err, int errlen);
/* The reference's own slow-step capture (run_step, attention.cpp:302-441):
 * tokens[0..n-2] through dense_attention_step without capture, then the last
 * token with CaptureSpec{window, allowed, pool, context}. Outputs (layer 0):
 * out_logits [H][nJ] (LogitWindow values), out_ctx [Hq*d] (attention context),
 * out_q [Hq*d] (the post-rotary query the step attended with, restated from
 * run_step's first lines: rmsnorm, wq, apply_rope — test infrastructure),
 * out_k / out_v [n][H*d] (the paged rows KvStore holds). */
int orc_toy_capture(const orc_toy_spec* spec, uint64_t seed, const int32_t* tokens, int n,
                    int nJ, const int32_t* allowed, int pool, double* out_logits, double* out_ctx,
                    double* out_q, float* out_k, float* out_v, char* err, int errlen);

#pragma GCC visibility pop
#ifdef __cplusplus
}
#endif

#endif

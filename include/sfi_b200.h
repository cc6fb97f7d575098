/*
 * sfi_b200.h — C ABI of the B200-native SFI decode-attention hot path.
 *
 * This is the drop-in boundary: plain pointers and sizes, int status codes,
 * no C++ or torch types. Every entry point is stream-ordered on the caller's
 * cudaStream_t (passed as void*), never synchronizes the host, and replaces a
 * reference CPU function (paths relative to /root/reference/proj):
 *
 *   sfi_ring_append     KvStore::append_layer            attention.cpp:136-152
 *                       + the recent window slide         scheduler.cpp:45-51
 *   sfi_dense_decode    attention_kernel_dense + the slow-step logit capture
 *                       attention.cpp:502-523, 80-113, 367-409
 *   sfi_selector        run_selector + stats_for_layer    selector.cpp:254-299,
 *                                                         scheduler.cpp:150-180
 *   sfi_compact_build   KvStore::reorganize               attention.cpp:186-217
 *   sfi_sparse_decode   attention_kernel_sparse           attention.cpp:525-550
 *   sfi_fast_decode     append_layer + sparse attention of one fast step
 *                       attention.cpp:354-360, 136-152, 270-291, 80-113
 *
 * Data layout (all device memory, caller-owned):
 *   k_cache, v_cache : bf16 [n_layers][batch][n_kv_heads][max_positions][head_dim]
 *                      row p-1 holds position p (1-based, distribution.hpp:23-26)
 *   key_norms        : fp64 [n_layers][batch][n_kv_heads][max_positions]
 *   ck, cv (compact) : bf16 [n_layers][batch][n_kv_heads][compact_rows][head_dim]
 *                      compact_rows = n_recent + n_sink + k_budget:
 *                      rows [0, n_recent)            recent ring, slot (p-1) % n_recent
 *                      rows [n_recent, +n_sink_b)    sink positions 1..n_sink_b
 *                      rows [.., +n_sel)             selected positions, ascending
 *   sel              : int32 [n_layers][batch][n_kv_heads][k_budget] (1-based, ascending)
 *   n_sel            : int32 [n_layers][batch][n_kv_heads]
 *   prefix_len       : int32 [batch]  L_b = positions 1..L_b live, current token included
 *   n_sink_b         : int32 [batch]  min(n_sink, prompt length) (scheduler.cpp:69)
 *   recent_len       : int32 [batch]  recent window length rl_b <= n_recent
 *   error_flags      : uint32 [1]     bit (1 << code) set by kernels on a contract
 *                                     violation; read with sfi_read_errors
 * The allowed set of a slow step is the contiguous range
 * J_b = [n_sink_b + 1, L_b - rl_b] with rl_b = recent_len[b], normally
 * clamp(L_b - n_sink_b, 0, n_recent) (scheduler.cpp:45-51, 81-91). Pooled logits are fp32 [batch][n_kv_heads][max_positions],
 * entry (b, h, p - (n_sink_b + 1)) for p in J_b.
 */
#ifndef SFI_B200_H
#define SFI_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define SFI_API __attribute__((visibility("default")))
#else
#define SFI_API
#endif

/* 0 = success; 1..10 = 1 + sfi::ErrorCode (error.hpp:23-34); >= 100 ABI-level. */
typedef enum {
  SFI_OK = 0,
  SFI_ERR_CONFIG = 1,
  SFI_ERR_EMPTY_SUPPORT = 2,
  SFI_ERR_SUPPORT_MISMATCH = 3,
  SFI_ERR_NON_FINITE_INPUT = 4,
  SFI_ERR_OVERLAP_VIOLATION = 5,
  SFI_ERR_STALE_COMPACT = 6,
  SFI_ERR_OUT_OF_RANGE = 7,
  SFI_ERR_BAD_WEIGHT_FILE = 8,
  SFI_ERR_CONTEXT_OVERFLOW = 9,
  SFI_ERR_IO = 10,
  SFI_ERR_CUDA = 100,
  SFI_ERR_UNSUPPORTED = 101,
  SFI_ERR_INVALID_ARGUMENT = 102
} sfi_status;

typedef enum { SFI_POOL_MEAN = 0, SFI_POOL_MAX = 1 } sfi_pool_mode; /* config.hpp:28 */

/* Static shape of one device cache (ModelSpec attention.hpp:31-44 + CacheLimits config.hpp:62-68). */
typedef struct {
  int32_t n_layers;
  int32_t batch;
  int32_t n_kv_heads;    /* H */
  int32_t n_q_heads;     /* Hq, multiple of H; group G = Hq / H in {1,2,4,8,16} */
  int32_t head_dim;      /* d in {64, 128} */
  int32_t max_positions; /* per-(layer, b, head) paged capacity */
  int32_t n_sink;        /* CacheLimits::n_sink */
  int32_t k_budget;      /* CacheLimits::k_budget == SelectorConfig::k_budget */
  int32_t n_recent;      /* CacheLimits::n_recent (ring capacity) */
} sfi_shape;

/* Device buffers of one cache (layout in the header comment). */
typedef struct {
  void* k_cache;
  void* v_cache;
  double* key_norms;
  void* ck;
  void* cv;
  int32_t* sel;
  int32_t* n_sel;
  int32_t* prefix_len;
  int32_t* n_sink_b;
  int32_t* recent_len; /* [batch] recent window length; sfi_step_advance keeps it at
                          clamp(L_b - n_sink_b, 0, n_recent) (scheduler.cpp:45-51) */
  uint32_t* error_flags;
  void* workspace; /* >= sfi_sizes.workspace (sfi_buffer_sizes); must be zeroed once at allocation */
  size_t workspace_bytes;
} sfi_cache;

/* Selector hyperparameters (SelectorConfig, config.hpp:31-47). k_budget comes from sfi_shape. */
typedef struct {
  double alpha, gamma, beta, p_curve, eta, lambda_clip, alpha_soft, alpha_cross,
      temperature, epsilon;
  int32_t nms_radius;
  int32_t pool; /* sfi_pool_mode; selects the pooling used by sfi_dense_decode */
} sfi_selector_params;

/* Byte sizes of every buffer for a shape (for the caller's allocator). */
typedef struct {
  size_t kv_cache;   /* each of k_cache, v_cache */
  size_t key_norms;
  size_t compact;    /* each of ck, cv */
  size_t sel;
  size_t n_sel;
  size_t per_batch;  /* prefix_len, n_sink_b */
  size_t workspace;
  size_t pooled_logits; /* fp32 [batch][n_kv][max_positions] */
} sfi_sizes;

SFI_API const char* sfi_version(void);
/* Thread-local message of the last non-OK status returned on this thread. */
SFI_API const char* sfi_last_error(void);
SFI_API int sfi_shape_validate(const sfi_shape* shape);
SFI_API int sfi_buffer_sizes(const sfi_shape* shape, sfi_sizes* out);
SFI_API void sfi_default_selector_params(sfi_selector_params* out);

/* Host-side recent window / allowed range for one request (scheduler.cpp:45-51, 81-91). */
SFI_API void sfi_recent_window(int32_t prefix_len, int32_t n_sink_b, int32_t n_recent,
                               int32_t* recent_start, int32_t* recent_len);

/* Host -> device per-request lengths: prefix_len[b], n_sink_b[b] and
 * recent_len[b] (NULL recent_len: the SFI rule clamp(L - n_sink_b, 0, n_recent)). */
SFI_API int sfi_set_lengths(const sfi_shape* shape, const sfi_cache* cache,
                            const int32_t* prefix_len_host, const int32_t* n_sink_host,
                            const int32_t* recent_len_host, void* stream);

/* prefix_len[b] += 1 for every request: opens the next decode step
 * (KvStore::begin_token attention.cpp:128-134; fast/slow_step_update
 * scheduler.cpp:101-131) and slides recent_len[b] by the SFI rule. Past
 * max_positions it sets SFI_ERR_CONTEXT_OVERFLOW and leaves prefix_len; until the
 * flags are read, sfi_ring_append and the fused sfi_fast_decode skip the append
 * (no valid row is overwritten). */
SFI_API int sfi_step_advance(const sfi_shape* shape, const sfi_cache* cache, void* stream);

/* Appends the current token (row prefix_len[b]-1) of `layer`:
 * k_new, v_new bf16 [batch][n_kv_heads][head_dim] -> paged cache, recent ring
 * slot (L_b-1) % n_recent, and the fp64 key norm sqrt(sum_c k_c^2) summed in
 * c order (attention.cpp:143-150). */
SFI_API int sfi_ring_append(const sfi_shape* shape, const sfi_cache* cache, int32_t layer,
                            const void* k_new, const void* v_new, void* stream);

/* Same for `count` consecutive positions starting at row prefix_len[b] (prefill;
 * does not move prefix_len): k, v bf16 [batch][n_kv_heads][count][head_dim]. */
SFI_API int sfi_append_block(const sfi_shape* shape, const sfi_cache* cache, int32_t layer,
                             int32_t count, const void* k, const void* v, void* stream);

/* Slow step, one layer: o = softmax(q K^T / sqrt(d)) V over positions
 * 1..L_b for every q head (fp32 accumulation over bf16 KV); when
 * pooled_logits != NULL also emits the raw logits q.k/sqrt(d) over J_b
 * pooled across each GQA group (mean or max, attention.cpp:394-409).
 * q, out: fp32 [batch][n_q_heads][head_dim]. */
SFI_API int sfi_dense_decode(const sfi_shape* shape, const sfi_cache* cache, int32_t layer,
                             const float* q, float* out, float* pooled_logits,
                             int32_t pool_mode, void* stream);

/* sfi_dense_decode with options. lse (optional): natural-log sum-exp per q head
 * (partial mode, see sequence sharding). flags: SFI_DENSE_SHARE_SM sizes the
 * stream-K grid to 65% of the SM slots (G <= 8; all of them at G = 16, where
 * the kernel is latency-bound) so kernels on another stream — the previous
 * layer's Selector in the asynchronous slow-step pipeline — run at the same
 * time on the rest. */
#define SFI_DENSE_SHARE_SM 2
/* Kernel choice for the dense decode (default: SFI_DENSE_TC env, else mma.sync):
 * SFI_DENSE_TC = the tcgen05/TMEM kernel (D = 128, G in {4, 8, 16}),
 * SFI_DENSE_MMA = the mma.sync kernel. */
#define SFI_DENSE_TC 4
#define SFI_DENSE_MMA 8
SFI_API int sfi_dense_decode_ex(const sfi_shape* shape, const sfi_cache* cache, int32_t layer,
                                const float* q, float* out, float* lse, float* pooled_logits,
                                int32_t pool_mode, int32_t flags, void* stream);

/* Fast step, one layer: attention over the compact cache only (ring + sink +
 * selected rows; S = recent_len + n_sink_b + n_sel per (b, head)). */
SFI_API int sfi_sparse_decode(const sfi_shape* shape, const sfi_cache* cache, int32_t layer,
                              const float* q, float* out, void* stream);

/* Fast step, one layer, ONE launch: sfi_ring_append of the current token
 * (k_new, v_new bf16 [batch][n_kv_heads][head_dim]; bit-identical paged row,
 * ring slot and key norm) fused with sfi_sparse_decode (the token attends to
 * itself, attention.cpp:354-360). flags: SFI_FAST_PREFETCH lets the kernel
 * stream this layer's compact rows before its programmatic-dependent-launch
 * wait — only valid when the kernel enqueued immediately before it on the
 * stream does not write this layer's compact rows, n_sel or n_sink_b (true for
 * every kernel of a fast step; false right after sfi_compact_build /
 * sfi_set_selection of the same layer). */
#define SFI_FAST_PREFETCH 1
SFI_API int sfi_fast_decode(const sfi_shape* shape, const sfi_cache* cache, int32_t layer,
                            const float* q, const void* k_new, const void* v_new, float* out,
                            int32_t flags, void* stream);

/* Selector, one layer: pooled logits over J_b (+ cached key norms) ->
 * sel/n_sel of `layer`, indices bit-exact with run_selector given identical
 * logits (fp64 arithmetic, (score desc, position asc) tie rule). */
SFI_API int sfi_selector(const sfi_shape* shape, const sfi_cache* cache, int32_t layer,
                         const float* pooled_logits, const sfi_selector_params* params,
                         void* stream);

/* Prefill tail-window capture (prefill_dense attention.cpp:460-500, capture
 * :367-409): for the W <= 16 window rows of every request — queries q fp32
 * [batch][W][n_q_heads][head_dim] at 1-based positions q_pos int32 [batch][W]
 * (device) — the raw logits q.k/sqrt(d) over J_b pooled across each GQA group
 * (mean or max), kMaskedLogit (-1e30) where the position is ahead of the row.
 * logits_out fp32 [batch][n_kv_heads][W][max_positions], entry (b, h, w, p - J_b.front()).
 * The cache holds the prompt (rows 1..L_b) and its lengths define J_b. */
SFI_API int sfi_prefill_capture(const sfi_shape* shape, const sfi_cache* cache, int32_t layer,
                                const float* q, int32_t W, const int32_t* q_pos, float* logits_out,
                                int32_t pool_mode, void* stream);
/* sfi_selector over a W-row window (logits [batch][n_kv_heads][W][max_positions]
 * as written by sfi_prefill_capture): evidence is the alpha power mean of the W
 * row softmaxes (evidence_from_window selector.cpp:96-127). */
SFI_API int sfi_selector_window(const sfi_shape* shape, const sfi_cache* cache, int32_t layer,
                                const float* logits, int32_t W, const sfi_selector_params* params,
                                void* stream);

/* KV-head-sharded Selector. Every Selector stage is
 * per head except cross-head exclusivity (selector.cpp:204-230), a softmax over
 * ALL kv heads of a request at each position. A rank whose cache holds heads
 * [shard * H, (shard + 1) * H) of n_shards * H (H = shape->n_kv_heads):
 *   1. sfi_selector_fuse: evidence, prior, fusion -> z_base of its heads in
 *      *z_local (device, inside the workspace; *z_bytes bytes, layout
 *      [batch][H][max_positions] fp64);
 *   2. all-gathers the z_local blocks of the n_shards ranks in rank order into
 *      z_all (n_shards * z_bytes; e.g. ncclAllGather on the same stream);
 *   3. sfi_selector_finish: soft-NMS and cross-head over all heads in global head
 *      order, top-k of its own heads -> sel / n_sel. Indices are bit-identical
 *      to the unsharded sfi_selector. */
SFI_API int sfi_selector_fuse(const sfi_shape* shape, const sfi_cache* cache, int32_t layer,
                              const float* pooled_logits, const sfi_selector_params* params,
                              const double** z_local, size_t* z_bytes, void* stream);
SFI_API int sfi_selector_finish(const sfi_shape* shape, const sfi_cache* cache, int32_t layer,
                                const sfi_selector_params* params, const double* z_all,
                                int32_t n_shards, int32_t shard, void* stream);

/* ---- Sequence sharding ------------------------------
 * Rank r of P holds positions (pos_base, pos_base + max_positions] of every
 * request (the last rank: everything from pos_base on; decode appends there).
 * The request's GLOBAL lengths live in caller-owned device arrays g_prefix_len,
 * g_n_sink, g_recent_len [batch]; sfi_seq_lengths (optionally advancing them
 * by `advance` first, like sfi_step_advance) rewrites the cache's own
 * prefix_len / n_sink_b / recent_len as this shard's LOCAL view (rows held,
 * sink rows at its start, recent rows at its end) and writes j_off[b] (global J
 * index of the shard's first J position) and n_glob[b] (global |J|). Every
 * single-GPU entry point then runs unchanged on the shard. */
SFI_API int sfi_seq_lengths(const sfi_shape* shape, const sfi_cache* cache, int32_t* g_prefix_len,
                            const int32_t* g_n_sink, int32_t* g_recent_len, int32_t advance,
                            int32_t pos_base, int32_t is_last, int32_t* j_off, int32_t* n_glob,
                            void* stream);
/* Partial attention of a shard: normalised O plus its natural-log sum-exp
 * lse fp32 [batch][n_q_heads]; a shard without rows gives O = 0, lse = -inf. */
SFI_API int sfi_dense_decode_partial(const sfi_shape* shape, const sfi_cache* cache, int32_t layer,
                                     const float* q, float* out, float* lse, float* pooled_logits,
                                     int32_t pool_mode, void* stream);
/* k_new / v_new NULL on shards that do not own the current position. */
SFI_API int sfi_fast_decode_partial(const sfi_shape* shape, const sfi_cache* cache, int32_t layer,
                                    const float* q, const void* k_new, const void* v_new, float* out,
                                    float* lse, int32_t flags, void* stream);
/* out[row] = sum_p exp(lse_p[row] - LSE[row]) o_p[row] in part order (the
 * all-gathered partials: o_parts [n_parts][rows][head_dim], lse [n_parts][rows]). */
SFI_API int sfi_merge_partials(int32_t n_parts, int32_t rows, int32_t head_dim, const float* o_parts,
                               const float* lse_parts, float* out, void* stream);

/* Peer-memory partial exchange (sequence sharding over NVLink P2P, no
 * collective launch): every rank maps every other rank's partial buffers and
 * epoch flag (CUDA IPC handles exchanged once).
 *   sfi_peer_publish: after the partial producer on `stream`, bumps this rank's
 *     flag (system-scope release).
 *   sfi_peer_merge: waits until every rank's flag reached this rank's own flag
 *     (acquire), then merges the n_parts partials read in place, in rank order
 *     (o_ptrs[i] fp32 [rows][head_dim], lse_ptrs[i] fp32 [rows]; device arrays of
 *     device pointers) — bit-identical to sfi_merge_partials on gathered copies.
 * A rank may rewrite a partial buffer once every rank has merged it: with one
 * buffer per layer (>= 2 layers) the stream order guarantees it. */
SFI_API int sfi_peer_publish(int32_t* flag, void* stream);
/* All-gather over the same protocol: dst[r] = rank r's `bytes`-byte block
 * (src_ptrs[r], device array of device pointers), read in place once rank r's
 * flag reached this rank's (bytes a multiple of 4). Used for the sequence-sharded
 * Selector's statistics, soft-NMS edges and top-k candidates. */
SFI_API int sfi_peer_gather(int32_t n_parts, int64_t bytes, const void* const* src_ptrs,
                            const int32_t* const* flag_ptrs, const int32_t* my_flag, void* dst, void* stream);
SFI_API int sfi_peer_merge(int32_t n_parts, int32_t rows, int32_t head_dim, const float* const* o_ptrs,
                           const float* const* lse_ptrs, const int32_t* const* flag_ptrs, const int32_t* my_flag,
                           float* out, void* stream);
/* Sequence-sharded Selector, decode path (W = 1, alpha = 1), per layer, three
 * exchanges:
 *   stats phase 1 -> row_stats [B*H][6]: local max and the five sums of
 *                    p = exp(v - local max), w, p^2, pw, w^2 ; all-gather -> stats_all
 *   stats phase 3 -> sums rescaled to the global max (shard order), p recomputed
 *                    as exp(v - global max) from the same logits, z_base + edges
 *                    [B*H][2R+2] (sfi_seq_edges_doubles) ; all-gather
 *   finish: soft-NMS with the neighbours' edges, cross-head (all heads local),
 *           local top-k -> candidates (z_adj, global position) [B*H][k_budget] ; all-gather
 *   pick: global top-k of the P candidate lists (shard order = position order,
 *         the reference's (score desc, position asc) rule) -> this shard's
 *         positions, local, into sel / n_sel.
 * Indices match the 1-GPU Selector (sums differ only in fp64 rounding order). */
SFI_API size_t sfi_seq_edges_doubles(const sfi_shape* shape, const sfi_selector_params* params);
SFI_API int sfi_seq_selector_stats(const sfi_shape* shape, const sfi_cache* cache, int32_t layer,
                                   const float* pooled_logits, const sfi_selector_params* params,
                                   const int32_t* j_off, const int32_t* n_glob, int32_t phase,
                                   double* row_stats, const double* stats_all, int32_t n_shards,
                                   double* edges, void* stream);
SFI_API int sfi_seq_selector_finish(const sfi_shape* shape, const sfi_cache* cache, int32_t layer,
                                    const sfi_selector_params* params, const int32_t* j_off,
                                    const int32_t* n_glob, const double* edges_all, int32_t n_shards,
                                    int32_t pos_base, double* cand_score, int32_t* cand_pos,
                                    void* stream);
SFI_API size_t sfi_seq_pick_scratch_bytes(const sfi_shape* shape, int32_t n_shards);
SFI_API int sfi_seq_selector_pick(const sfi_shape* shape, const sfi_cache* cache, int32_t layer,
                                  int32_t n_shards, const double* cand_score_all,
                                  const int32_t* cand_pos_all, int32_t pos_base, int32_t pos_end,
                                  void* scratch, void* stream);

/* ---- Multi-GPU over an NCCL communicator (SURVEY §8b "a multi-GPU variant
 * taking an NCCL communicator", §8e) -----------------------------------------
 * `nccl_comm` is an ncclComm_t (ncclCommInitRank, or the communicator of
 * torch's ProcessGroupNCCL) of the n_shards ranks; every call enqueues its
 * kernels and the ncclAllGather calls on `stream`, no host sync (graph
 * capturable). NCCL is resolved at run time from the process (the library
 * that created the communicator); SFI_ERR_UNSUPPORTED when none is loaded.
 *   sfi_selector_sharded_nccl  C3 KV-head sharding: sfi_selector_fuse, the
 *       z_base all-gather into z_all [n_shards][B][H][max_positions] fp64,
 *       sfi_selector_finish (cross-head over all heads, top-k of own heads) —
 *       indices bit-identical to the unsharded Selector (cross-head coupling,
 *       selector.cpp:204-230).
 *   sfi_merge_partials_nccl    C4 sequence sharding: all-gather of this rank's
 *       (O, LSE) partials (o_part [rows][head_dim], lse_part [rows]) into
 *       o_all / lse_all, then sfi_merge_partials in rank order.
 *   sfi_seq_selector_nccl      C4: the sharded Selector's three exchanges (row
 *       statistics, soft-NMS edges, top-k candidates) and the global pick;
 *       scratch of sfi_seq_selector_nccl_scratch_bytes. */
SFI_API int sfi_selector_sharded_nccl(const sfi_shape* shape, const sfi_cache* cache, int32_t layer,
                                      const float* pooled_logits, const sfi_selector_params* params,
                                      void* nccl_comm, int32_t n_shards, int32_t shard, double* z_all, void* stream);
SFI_API int sfi_merge_partials_nccl(int32_t n_parts, int32_t rows, int32_t head_dim, const float* o_part,
                                    const float* lse_part, float* o_all, float* lse_all, float* out,
                                    void* nccl_comm, void* stream);
SFI_API size_t sfi_seq_selector_nccl_scratch_bytes(const sfi_shape* shape, const sfi_selector_params* params,
                                                   int32_t n_shards);
SFI_API int sfi_seq_selector_nccl(const sfi_shape* shape, const sfi_cache* cache, int32_t layer,
                                  const float* pooled_logits, const sfi_selector_params* params,
                                  const int32_t* j_off, const int32_t* n_glob, int32_t pos_base, int32_t pos_end,
                                  void* nccl_comm, int32_t n_shards, void* scratch, size_t scratch_bytes,
                                  void* stream);

/* Measurement aid: n_launches empty kernels of `grid` CTAs with the fused fast
 * step's programmatic-dependent-launch protocol, back to back on `stream` — the
 * per-layer launch floor a one-launch-per-layer fast step cannot go below. */
SFI_API int sfi_launch_floor(int32_t n_launches, int32_t grid, void* stream);

/* run_selector on explicit device arrays (the reference-facing form,
 * selector.cpp:254-299): H heads, a W x n window per head over an arbitrary
 * ascending allowed list. logits fp64 [H][W][n], norms fp64 [H][n] (CacheStats
 * key norms), allowed int32 [n]; scratch >= sfi_selector_explicit_scratch_bytes;
 * outputs sel int32 [H][k_budget] ascending, n_sel int32 [H]; contract
 * violations set bits in err (uint32 device word). W <= 16, H <= 16. */
SFI_API size_t sfi_selector_explicit_scratch_bytes(int32_t H, int32_t n);
SFI_API int sfi_selector_explicit(int32_t H, int32_t W, int32_t n, int32_t k_budget,
                                  const double* logits, const double* norms,
                                  const int32_t* allowed, const sfi_selector_params* params,
                                  void* scratch, int32_t* sel, int32_t* n_sel, uint32_t* err,
                                  void* stream);

/* select_top_k (selector.cpp:232-252) on device arrays: rows independent score
 * rows fp64 [rows][n] over allowed int32 [n]; sel int32 [rows][k], n_sel [rows]. */
SFI_API int sfi_select_top_k(int32_t rows, int32_t n, int32_t k, const double* scores,
                             const int32_t* allowed, int32_t* sel, int32_t* n_sel, void* stream);

/* Selector stages, one at a time (the reference's stage API: evidence_from_window
 * selector.cpp:96-127, prior_from_stats :129-160, fuse :162-185, z = log(s+eps)
 * :270-276, refine_soft_nms :187-202, refine_cross_head :204-230, normalize
 * distribution.cpp:41-60). Device arrays, fp64, one row per head:
 *   EVIDENCE    a = logit window [H][W*n]            -> out = f [H][n]
 *   PRIOR       a = key norms [H][n], b = u(j) [n]    -> out = r [H][n]
 *   NORMALIZE   a = weights [H][n]                   -> out [H][n]
 *   FUSE        a = f [H][n], b = r [H][n]           -> out = s [H][n], out2 = lambda* [H]
 *   Z_BASE      a = s [H][n]                         -> out = log(s + eps)
 *   SOFT_NMS    a = z [H][n] (rank-order rows)       -> out [H][n]
 *   CROSS_HEAD  a = z [H][n]                         -> out [H][n]
 * head_err [H] int32 (EVIDENCE / PRIOR / NORMALIZE): 0, or the sfi_status of
 * the head's first failure in the reference's check order; the caller zeroes
 * it and reads it after the stream. Stream-ordered, no host sync. */
#define SFI_STAGE_EVIDENCE 0
#define SFI_STAGE_PRIOR 1
#define SFI_STAGE_NORMALIZE 2
#define SFI_STAGE_FUSE 3
#define SFI_STAGE_Z_BASE 4
#define SFI_STAGE_SOFT_NMS 5
#define SFI_STAGE_CROSS_HEAD 6
SFI_API int sfi_selector_stage(int32_t stage, int32_t H, int32_t W, int32_t n, const double* a, const double* b,
                               const sfi_selector_params* params, double* out, double* out2, int32_t* head_err,
                               void* stream);

/* Debug: after sfi_selector, copies the fp64 stage arrays z_base and z_adj
 * (selector.cpp:270-297) of request b into host buffers [n_kv_heads][n_J]. */
SFI_API int sfi_selector_stages(const sfi_shape* shape, const sfi_cache* cache, int32_t b,
                                double* z_base, double* z_adj, int32_t n_j, void* stream);

/* Compact-cache builder, one layer: gathers sink rows and selected rows
 * (sel/n_sel of `layer`) into the compact buffer; with rebuild_ring also
 * refills the recent ring from the paged cache. Validates strictly ascending
 * merged positions within [1, L_b] (kOverlapViolation / kOutOfRange). */
SFI_API int sfi_compact_build(const sfi_shape* shape, const sfi_cache* cache, int32_t layer,
                              int32_t rebuild_ring, void* stream);

/* Host-supplied selection for one layer (KvStore::reorganize semantics):
 * sel_host int32 [batch][n_kv_heads][k_budget], counts [batch][n_kv_heads];
 * copied to the device, then sfi_compact_build. Synchronous on `stream`. */
SFI_API int sfi_set_selection(const sfi_shape* shape, const sfi_cache* cache, int32_t layer,
                              const int32_t* sel_host, const int32_t* counts_host,
                              void* stream);

/* Reads (and clears) the device error word; synchronizes `stream`. Returns
 * the lowest set code as the status (SFI_OK when clean). */
SFI_API int sfi_read_errors(const sfi_cache* cache, uint32_t* flags_out, void* stream);

/* Deterministic synthetic bf16 N(0,~1) fill of the paged cache rows [0, len)
 * of every (layer, b, head) plus their key norms (bench / tests only). */
SFI_API int sfi_fill_synthetic(const sfi_shape* shape, const sfi_cache* cache, uint64_t seed,
                               int32_t len, void* stream);

/* Number of kernels the last call on this thread enqueued (launch accounting). */
SFI_API int32_t sfi_last_launch_count(void);

/* Debug (tuning): with SFI_DECODE_TRACE set in the environment, copies the
 * per-CTA timeline of the last decode launch ([ctas][8] int64: start ns,
 * prologue done, first tile landed, end, emissions, tiles, smid) into `out`;
 * returns the CTA count. SFI_DECODE_CTAS=<n> overrides the decode grid. */
SFI_API int32_t sfi_debug_decode_trace(int64_t* out, int32_t max_ctas);
/* Debug: with SFI_LAYER_TRACE set, every fast-step launch keeps its per-CTA
 * timeline in a slot of its layer (no reset); copies [layers][max_ctas][16]
 * int64 into `out` and returns the CTA count of the last launch. */
SFI_API int32_t sfi_debug_layer_trace(int64_t* out, int32_t layers, int32_t max_ctas);

#ifdef __cplusplus
}
#endif

#endif /* SFI_B200_H */

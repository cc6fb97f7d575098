// selector.cu — K2: the SFI Selector on the device, fp64 end to end.
//
// Reference (paths relative to /root/reference/proj):
//   make_cache_stats     selector.cpp:78-94    u = (j - j_min) / ((j_max - j_min) + eps)
//   row_softmax          selector.cpp:54-74    p = exp(v - max), max from kMaskedLogit
//   evidence_from_window selector.cpp:96-127   power mean over W rows, normalize
//   prior_from_stats     selector.cpp:129-160  (|k|+eps)^-g exp(-b u^p) (1-u+eps)^eta
//   normalize            distribution.cpp:41-60
//   fuse                 selector.cpp:162-185  lambda* closed form, clip
//   z = log(s + eps)     selector.cpp:270-276
//   refine_soft_nms      selector.cpp:187-202
//   refine_cross_head    selector.cpp:204-230
//   select_top_k         selector.cpp:232-252  (score desc, position asc)
//
// Three kernels per call:
//   sel_fuse_*        one 8-CTA cluster per (b, head) row. Decode fast path
//                     (W = 1, alpha = 1): pass 1 row max; pass 2 p = exp(v-max)
//                     and the prior weight w with the five sums
//                     sum p, sum w, sum p^2, sum pw, sum w^2 in ONE cluster
//                     reduction (f = p/sum p and r = w/sum w are rescalings,
//                     so |f|^2, f.r, |r|^2 follow from them); pass 3 z_base.
//                     The general path (W > 1 or alpha != 1) keeps the
//                     reference's pass structure.
//   sel_refine_kernel 256 positions of one request per CTA, all heads staged
//                     in shared memory with the NMS halo; soft-NMS per head,
//                     then the cross-head softmax in head order with
//                     log r_h = (z_h - max)/T - log(sum) (one log per position).
//   sel_topk_kernel   one 8-CTA cluster per row, the row's 64-bit
//                     order-preserving keys resident in shared memory: exact
//                     K-th key by radix refinement (11-bit digits, histograms
//                     merged over DSMEM, 2 cluster barriers per digit), then an
//                     ordered cluster scan emits the selected positions
//                     ascending with the reference tie rule (equal scores ->
//                     lower position).
// The production decode path (cache mode, W = 1, alpha = 1, unsharded) instead
// runs sel_pw (chunk statistics + prior weights) -> sel_coef (row max M,
// lambda*, coefficients) -> sel_z (z_base, soft-NMS, cross-head -> z_adj) and
// then the single-CTA top-k (|J| <= 48K: sel_topk_cta_kernel) or, for long
// rows, the rows x segments histogram top-k (sel_bt_thresh / scan / emit).
// Inputs come either from the device cache (production: fp32 pooled logits
// over the contiguous J_b, cached fp64 key norms) or from explicit arrays
// (reference-facing run_selector: fp64 W x |J| windows over an arbitrary
// ascending allowed list).
// Compiled with -fmad=false (no FMA contraction). Reductions are tree-ordered
// and the fast path rescales instead of dividing twice, so intermediates can
// differ from the reference by a few ulps (~1e-16 relative). The index
// contract: every score is a deterministic function of the same inputs the
// reference's score is a function of (p from the ROW max, never a chunk max),
// so exact ties in the reference are exact ties here and resolve the same way
// (lower position first); strict orderings agree whenever the K-th/(K+1)-th
// gap exceeds a few ulps — measured >= 3.7e-8 relative.
// Checked by tests/test_gpu_parity.py and tests/test_baseline_parity.py
// (full BASELINE layers, forced ties across statistics chunks).
#include <cooperative_groups.h>

#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace cg = cooperative_groups;

namespace sfi_impl {

using namespace sfi_dev;

namespace {

constexpr int kCS = 8;      // CTAs per cluster
constexpr int kT = 512;     // threads per CTA
constexpr int kWarps = kT / 32;
constexpr int kBins = 2048; // 11-bit radix digits
constexpr int kBinsPerCta = kBins / kCS;
constexpr int kMaxW = 16;   // observation window rows (prefill window_prefill = 16)
constexpr int kRefineT = 256;
constexpr int kMaxNmsR = 16;  // smem halo of the refine kernel
constexpr int kTopkSmemKeys = 22 * 1024;  // keys per CTA kept in shared memory
constexpr int kCandCap = 512;             // threshold-bucket size resolved by direct ranking
constexpr double kMaskedLogit = -1e30;  // selector.hpp:42

struct SelParams {
  // cache mode
  const float* logits32;    // [rows][W][ld] fp32
  const double* norms_c;    // this layer's cache norms: [rows][Lmax] by position
  const int32_t* prefix_len;
  const int32_t* n_sink_b;
  const int32_t* recent_len;
  // explicit mode
  const double* logits64;   // [rows][W][ld]
  const double* norms_e;    // [rows][ld]
  const int32_t* allowed;   // [n] ascending
  int n_fixed;
  // common
  int W;
  int ld;                   // row stride of scratch / explicit arrays
  double* sa;               // [rows][ld]
  double* sb;               // [rows][ld]
  int32_t* sel;             // [rows][K]
  int32_t* n_sel;           // [rows]
  uint32_t* err;
  int B, H, Lmax, K;
  double alpha, gamma, beta, p_curve, eta, lambda_clip, alpha_soft, alpha_cross, temperature, eps;
  int nms_radius;
  // KV-head sharding: z_base of all H_all heads gathered
  // [n_shards][B][H][ld] (H = this shard's heads [h_off, h_off + H)); null = local
  const double* z_all;
  int H_all, h_off;
  // sequence sharding: this shard's J is the slice
  // [j_off[b], j_off[b] + n) of the global J of n_glob[b] positions
  const int32_t* j_off;
  const int32_t* n_glob;
  int seq_phase;            // 1 = local statistics, 3 = z_base + edges (0 = unsharded)
  double* row_stats;        // [rows][6] this shard's (max, sum p, sum w, sum p^2, sum pw, sum w^2),
                            //   p relative to the local max (phase 1 out, phase 3 in)
  const double* stats_all;  // [n_shards][rows][6] all-gathered row_stats (phase 3 in)
  double* edges;            // [rows][2R+2] (phase 3 out): first R, last R z_base values, j_off, n
  const double* edges_all;  // [n_shards][rows][2R+2] all-gathered edges (refine halo)
  int n_shards;
  // long-row top-k: sel_z adds every z_adj to a per-row value histogram
  uint32_t* bt_hist;        // [rows][kBtBins] or null
  double bt_zlo, bt_scale;  // bin = clamp((z - zlo) * scale)
};

// Row geometry: n = |J|, j_min, position of index j, u(j).
template <bool kExp>
struct Src {
  const SelParams& p;
  int n, j_min, b_;
  __device__ __forceinline__ Src(const SelParams& pp, int b) : p(pp), b_(b) {
    if (kExp) {
      n = p.n_fixed;
      j_min = n > 0 ? p.allowed[0] : 0;
    } else {
      const int L = p.prefix_len[b];
      const int nsb = p.n_sink_b[b];
      j_min = nsb + 1;
      n = max(0, (L - p.recent_len[b]) - j_min + 1);
    }
  }
  __device__ __forceinline__ double logit(int row, int w, int j) const {
    if (kExp) return p.logits64[((size_t)row * p.W + w) * p.ld + j];
    return (double)p.logits32[((size_t)row * p.W + w) * p.ld + j];
  }
  __device__ __forceinline__ double norm(int row, int j) const {
    if (kExp) return p.norms_e[(size_t)row * p.ld + j];
    return p.norms_c[(size_t)row * p.Lmax + (j_min - 1) + j];
  }
  // make_cache_stats: (double)(allowed[i] - j_min) / ((double)(j_max - j_min) + eps)
  __device__ __forceinline__ double u(int j, double denom) const {
    if (kExp) return (double)(p.allowed[j] - j_min) / denom;
    if (p.j_off) return (double)(j + p.j_off[b_]) / denom;  // global J index (sequence shard)
    return (double)j / denom;
  }
  __device__ __forceinline__ double u_denom() const {
    if (kExp) return (double)(p.allowed[n - 1] - j_min) + p.eps;
    if (p.n_glob) return (double)(p.n_glob[b_] - 1) + p.eps;
    return (double)(n - 1) + p.eps;
  }
  __device__ __forceinline__ int pos(int j) const { return kExp ? p.allowed[j] : j_min + j; }
};

// std::max semantics (first argument on ties)
__device__ __forceinline__ double smax(double a, double b) { return (a < b) ? b : a; }

// pow with the exponents the defaults use evaluated exactly (correctly
// rounded), everything else through CUDA's pow.
__device__ __forceinline__ double pow_ref(double x, double y) {
  if (y == 1.0) return x;
  if (y == 2.0) return x * x;
  if (y == 0.5) return sqrt(x);
  if (y == -1.0) return 1.0 / x;
  if (y == 0.0) return 1.0;
  return pow(x, y);
}

// prior_from_stats weight (selector.cpp:150-153)
__device__ __forceinline__ double prior_w(const SelParams& p, double norm, double u) {
  const double pi_kn = pow_ref(norm + p.eps, -p.gamma);
  const double pi_pos = exp(-p.beta * pow_ref(u, p.p_curve)) * pow_ref(1.0 - u + p.eps, p.eta);
  return pi_kn * pi_pos;
}

struct OpSum {
  __device__ double operator()(double a, double b) const { return a + b; }
};
struct OpMax {
  __device__ double operator()(double a, double b) const { return smax(a, b); }
};
struct OpMinU {
  __device__ unsigned long long operator()(unsigned long long a, unsigned long long b) const {
    return a < b ? a : b;
  }
};

// Deterministic cluster-wide reduction of the first `nv` of NV values: warp
// butterfly, warps in index order, CTAs in rank order; every thread of the
// cluster gets the same result. `red` is a [2][NV] buffer whose halves are
// used alternately by successive calls (`parity`; every call site of a kernel
// shares one buffer of the kernel's widest NV), so one cluster barrier per
// call suffices; the kernel ends with a cluster barrier before any CTA exits.
template <int NV, int S, typename T, typename Op>
__device__ __forceinline__ void cluster_reduce(T (&v)[NV], int nv, T* wbuf, T (*red)[S], int& parity,
                                               cg::cluster_group& cl, Op op) {
  static_assert(NV <= S, "reduction buffer too narrow");
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  T* slot = red[parity];
  parity ^= 1;
#pragma unroll
  for (int k = 0; k < NV; ++k)
    if (k < nv)
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v[k] = op(v[k], __shfl_xor_sync(0xffffffffu, v[k], o));
  if (lane == 0)
#pragma unroll
    for (int k = 0; k < NV; ++k)
      if (k < nv) wbuf[warp * NV + k] = v[k];
  __syncthreads();
  if (threadIdx.x < nv) {
    const int k = threadIdx.x;
    T acc = wbuf[k];
    for (int w = 1; w < kWarps; ++w) acc = op(acc, wbuf[w * NV + k]);
    slot[k] = acc;
  }
  cl.sync();
#pragma unroll
  for (int k = 0; k < NV; ++k)
    if (k < nv) {
      T acc = *cl.map_shared_rank(&slot[k], 0);
      for (int r = 1; r < (int)cl.num_blocks(); ++r) acc = op(acc, *cl.map_shared_rank(&slot[k], r));
      v[k] = acc;
    }
}

// Sequence shard: the soft-NMS halo its neighbours need — the first and last
// R z_base values of its J slice, then (j_off, n) — NaN where absent.
template <bool kExp>
__device__ __forceinline__ void write_edges(const SelParams& p, int row, const double* A, int n,
                                            const Src<kExp>& src) {
  const int R = p.nms_radius;
  const int w = 2 * R + 2;
  double* e = p.edges + (size_t)row * w;
  for (int t = threadIdx.x; t < w; t += blockDim.x) {
    double v;
    if (t < R) v = (t < n) ? A[t] : __longlong_as_double(0x7ff8000000000000ll);
    else if (t < 2 * R) {
      const int i = n - R + (t - R);
      v = (i >= 0 && i < n) ? A[i] : __longlong_as_double(0x7ff8000000000000ll);
    } else if (t == 2 * R) v = (double)(p.j_off ? p.j_off[src.b_] : 0);
    else v = (double)n;
    e[t] = v;
  }
}

// ---------------------------------------------------------------------------
// Stage A, decode fast path: W = 1, alpha = 1.
template <bool kExp>
__global__ void __cluster_dims__(kCS, 1, 1) __launch_bounds__(kT, 2)
    sel_fuse_fast_kernel(const SelParams p) {
  griddep_wait();  // PDL: logits come from the preceding dense decode
  griddep_launch();
  __shared__ double wbuf[kWarps * 5];
  __shared__ double red[2][5];
  cg::cluster_group cl = cg::this_cluster();
  const int rank = (int)cl.block_rank();
  const int row = blockIdx.y;
  const Src<kExp> src(p, row / p.H);
  const int n = src.n;
  const int ph = p.seq_phase;
  if (n <= 0) {  // uniform over the cluster
    if (ph != 0 && rank == 0) {  // sequence shard without J positions: neutral stats
      if (ph == 1 && threadIdx.x < 6) p.row_stats[row * 6 + threadIdx.x] = threadIdx.x == 0 ? kMaskedLogit : 0.0;
      if (ph == 3) write_edges(p, row, nullptr, 0, src);
    }
    return;
  }
  const int chunk = (n + kCS - 1) / kCS;
  const int lo = rank * chunk;
  const int hi = min(n, lo + chunk);
  double* A = p.sa + (size_t)row * p.ld;
  double* Bw = p.sb + (size_t)row * p.ld;
  int par = 0;

  // pass 1: row max (starts at kMaskedLogit), finite check
  double m1[1] = {kMaskedLogit};
  if (ph == 3) goto after_max;  // sequence shard: w and the statistics come from phase 1
  {
  bool bad = false;
  for (int j = lo + threadIdx.x; j < hi; j += kT) {
    const double v = src.logit(row, 0, j);
    if (!isfinite(v)) bad = true;
    m1[0] = smax(m1[0], v);
  }
  if (bad) raise_error(p.err, SFI_ERR_NON_FINITE_INPUT);
  cluster_reduce<1>(m1, 1, wbuf, red, par, cl, OpMax());
  }
after_max:
  // (phase 3 of a sequence shard: this shard's local max from its phase 1)
  const double mx = ph == 3 ? p.row_stats[row * 6] : m1[0];

  // pass 2: p, w and the five sums
  const double denom_u = src.u_denom();
  double s[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
  bool badn = false;
  constexpr int kU = 2;  // loads of kU iterations are issued before any use
  // (a sequence shard's phase 3 reuses the w of its phase 1)
  for (int j0 = (ph == 3 ? hi : lo + threadIdx.x); j0 < hi; j0 += kU * kT) {
    double vv[kU], nn[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int j = j0 + u * kT;
      vv[u] = j < hi ? src.logit(row, 0, j) : 0.0;
      nn[u] = j < hi ? src.norm(row, j) : 1.0;
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int j = j0 + u * kT;
      if (j >= hi) break;
      const double v = vv[u];
      const double pj = (v <= kMaskedLogit) ? 0.0 : exp(v - mx);
      const double norm = nn[u];
      if (!isfinite(norm) || norm < 0.0) badn = true;
      const double wr = prior_w(p, norm, src.u(j, denom_u));
      if (!isfinite(wr) || wr < 0.0) badn = true;
      A[j] = pj;
      Bw[j] = wr;
      s[0] += pj;
      s[1] += wr;
      s[2] += pj * pj;
      s[3] += pj * wr;
      s[4] += wr * wr;
    }
  }
  if (badn) raise_error(p.err, SFI_ERR_NON_FINITE_INPUT);
  double mg = mx;  // the global row max (sequence shard: the max over the gathered local maxima)
  if (ph == 3) {
    // the shards' statistics, rescaled to the global row max in shard order
    const int rows = p.B * p.H;
    double M = kMaskedLogit;
    for (int sh = 0; sh < p.n_shards; ++sh) M = smax(M, p.stats_all[((size_t)sh * rows + row) * 6]);
#pragma unroll
    for (int k = 0; k < 5; ++k) s[k] = 0.0;
    for (int sh = 0; sh < p.n_shards; ++sh) {
      const double* x = p.stats_all + ((size_t)sh * rows + row) * 6;
      const double e = exp(x[0] - M);
      s[0] += x[1] * e;
      s[1] += x[2];
      s[2] += x[3] * (e * e);
      s[3] += x[4] * e;
      s[4] += x[5];
    }
    mg = M;
  } else {
    cluster_reduce<5>(s, 5, wbuf, red, par, cl, OpSum());
  }
  if (ph == 1) {
    if (rank == 0 && threadIdx.x < 6) p.row_stats[row * 6 + threadIdx.x] = threadIdx.x == 0 ? mx : s[threadIdx.x - 1];
    cl.sync();
    return;
  }
  if (threadIdx.x == 0 && rank == 0 && (s[0] <= 0.0 || s[1] <= 0.0))
    raise_error(p.err, SFI_ERR_EMPTY_SUPPORT);
  // f = p c1, r = w c2 (normalize); fuse (selector.cpp:166-174)
  const double c1 = 1.0 / s[0], c2 = 1.0 / s[1];
  const double ff = s[2] * c1 * c1;
  const double fr = s[3] * c1 * c2;
  const double rr = s[4] * c2 * c2;
  const double denom = ff - 2.0 * fr + rr;
  double lambda = 0.0;
  if (fabs(denom) >= p.eps) {
    lambda = (ff - fr) / denom;
    lambda = (lambda < 0.0) ? 0.0 : (p.lambda_clip < lambda) ? p.lambda_clip : lambda;
  }
  const double a = (1.0 - lambda) * c1, bb = lambda * c2;

  // pass 3: z = log((1 - lambda) f + lambda r + eps)
  for (int j0 = lo + threadIdx.x; j0 < hi; j0 += kU * kT) {
    double pa[kU], wb[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int j = j0 + u * kT;
      if (ph == 3) {  // p = exp(v - global max), the same bits as the unsharded pass 2
        const double v = j < hi ? src.logit(row, 0, j) : kMaskedLogit;
        pa[u] = (v <= kMaskedLogit) ? 0.0 : exp(v - mg);
      } else {
        pa[u] = j < hi ? A[j] : 0.0;
      }
      wb[u] = j < hi ? Bw[j] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int j = j0 + u * kT;
      if (j < hi) A[j] = log(a * pa[u] + bb * wb[u] + p.eps);
    }
  }
  if (ph == 3) {
    cl.sync();  // every CTA's z_base written
    if (rank == 0) write_edges(p, row, A, n, src);
  }
  cl.sync();  // remote reads of `red` done before any CTA exits
}

// Stage A, general path (W >= 1, any alpha): the reference's pass structure.
template <bool kExp, int WM>
__global__ void __cluster_dims__(kCS, 1, 1) __launch_bounds__(kT)
    sel_fuse_kernel(const SelParams p) {
  griddep_wait();
  griddep_launch();
  constexpr int kNV = (WM + 1) > 3 ? (WM + 1) : 3;
  __shared__ double wbuf[kWarps * kNV];
  __shared__ double red[2][kNV];
  cg::cluster_group cl = cg::this_cluster();
  const int rank = (int)cl.block_rank();
  const int row = blockIdx.y;
  const Src<kExp> src(p, row / p.H);
  const int n = src.n;
  if (n <= 0) return;  // uniform over the cluster
  const int W = WM == 1 ? 1 : p.W;
  const int chunk = (n + kCS - 1) / kCS;
  const int lo = rank * chunk;
  const int hi = min(n, lo + chunk);
  double* A = p.sa + (size_t)row * p.ld;
  double* Bw = p.sb + (size_t)row * p.ld;
  int par = 0;

  // pass 1: per window row max (row_softmax: starts at kMaskedLogit), finite check
  double mx[WM];
#pragma unroll
  for (int w = 0; w < WM; ++w) mx[w] = kMaskedLogit;
  bool bad = false;
  for (int j = lo + threadIdx.x; j < hi; j += kT) {
#pragma unroll
    for (int w = 0; w < WM; ++w)
      if (w < W) {
        const double v = src.logit(row, w, j);
        if (!isfinite(v)) bad = true;
        mx[w] = smax(mx[w], v);
      }
  }
  if (bad) raise_error(p.err, SFI_ERR_NON_FINITE_INPUT);
  cluster_reduce<WM>(mx, W, wbuf, red, par, cl, OpMax());

  // pass 2: sum_j exp(v - max) per window row; prior weight w and its sum
  const double denom_u = src.u_denom();
  double s2[WM + 1];
#pragma unroll
  for (int k = 0; k <= WM; ++k) s2[k] = 0.0;
  bool badn = false;
  for (int j = lo + threadIdx.x; j < hi; j += kT) {
#pragma unroll
    for (int w = 0; w < WM; ++w)
      if (w < W) {
        const double v = src.logit(row, w, j);
        const double pj = (v <= kMaskedLogit) ? 0.0 : exp(v - mx[w]);
        if (WM == 1) A[j] = pj;
        s2[w] += pj;
      }
    const double norm = src.norm(row, j);
    if (!isfinite(norm) || norm < 0.0) badn = true;
    const double wr = prior_w(p, norm, src.u(j, denom_u));
    if (!isfinite(wr) || wr < 0.0) badn = true;
    Bw[j] = wr;
    s2[WM] += wr;
  }
  if (badn) raise_error(p.err, SFI_ERR_NON_FINITE_INPUT);
  s2[W] = s2[WM];  // pack the prior sum right after the W row sums
  cluster_reduce<WM + 1>(s2, W + 1, wbuf, red, par, cl, OpSum());
  const double sumw = s2[W];
  if (threadIdx.x == 0 && rank == 0) {
    for (int w = 0; w < W; ++w)
      if (s2[w] <= 0.0) raise_error(p.err, SFI_ERR_EMPTY_SUPPORT);
    if (sumw <= 0.0) raise_error(p.err, SFI_ERR_EMPTY_SUPPORT);
  }

  // pass 3: p /= sum; mu += pow(p, alpha) over rows; weight = pow(mu / W, 1/alpha)
  const bool a_one = (p.alpha == 1.0);
  const double inv_a = 1.0 / p.alpha;
  const double inv_w = 1.0 / (double)W;
  double s3[1] = {0.0};
  for (int j = lo + threadIdx.x; j < hi; j += kT) {
    double wt;
    if (WM == 1) {
      const double f1 = A[j] / s2[0];
      wt = a_one ? f1 : pow_ref((0.0 + pow_ref(f1, p.alpha)) * inv_w, inv_a);
    } else {
      double mu = 0.0;
      for (int w = 0; w < W; ++w) {
        const double v = src.logit(row, w, j);
        const double pj = ((v <= kMaskedLogit) ? 0.0 : exp(v - mx[w])) / s2[w];
        mu += pow_ref(pj, p.alpha);
      }
      wt = pow_ref(mu * inv_w, inv_a);
    }
    A[j] = wt;
    s3[0] += wt;
  }
  cluster_reduce<1>(s3, 1, wbuf, red, par, cl, OpSum());
  const double sum2 = s3[0];
  if (threadIdx.x == 0 && rank == 0 && sum2 <= 0.0) raise_error(p.err, SFI_ERR_EMPTY_SUPPORT);

  // pass 4: f = normalize(evidence), r = normalize(prior); |f|^2, f.r, |r|^2
  double s4[3] = {0.0, 0.0, 0.0};
  for (int j = lo + threadIdx.x; j < hi; j += kT) {
    const double f = A[j] / sum2;
    const double r = Bw[j] / sumw;
    A[j] = f;
    Bw[j] = r;
    s4[0] += f * f;
    s4[1] += f * r;
    s4[2] += r * r;
  }
  cluster_reduce<3>(s4, 3, wbuf, red, par, cl, OpSum());
  const double ff = s4[0], fr = s4[1], rr = s4[2];
  const double denom = ff - 2.0 * fr + rr;
  double lambda = 0.0;
  if (fabs(denom) >= p.eps) {
    lambda = (ff - fr) / denom;
    lambda = (lambda < 0.0) ? 0.0 : (p.lambda_clip < lambda) ? p.lambda_clip : lambda;
  }

  // pass 5: s = (1 - lambda) f + lambda r; z = log(s + eps)
  for (int j = lo + threadIdx.x; j < hi; j += kT) {
    const double s = (1.0 - lambda) * A[j] + lambda * Bw[j];
    A[j] = log(s + p.eps);
  }
  cl.sync();
}

// z_base row of (request b, global head h): local scratch, or the all-gathered
// [n_shards][B][H][ld] block of the head-sharded Selector
__device__ __forceinline__ const double* zrow(const SelParams& p, int b, int h) {
  if (p.z_all) return p.z_all + ((size_t)((h / p.H) * p.B + b) * p.H + (h % p.H)) * p.ld;
  return p.sa + (size_t)(b * p.H + h) * p.ld;
}

// z_base at global J index g from the all-gathered shard edges (first / last R
// values of every shard's slice, then its j_off and n)
__device__ __forceinline__ double halo(const SelParams& p, int row, int g, int R) {
  const int w = 2 * R + 2;
  const int rows = p.B * p.H;
  for (int s = 0; s < p.n_shards; ++s) {
    const double* e = p.edges_all + ((size_t)s * rows + row) * w;
    const int so = (int)e[2 * R], sn = (int)e[2 * R + 1];
    if (g >= so && g < so + sn) {
      const int li = g - so;
      return li < R ? e[li] : e[R + li - (sn - R)];
    }
  }
  return 0.0;  // unreachable for a consistent shard layout
}

// refine_cross_head (selector.cpp:204-230) at one position over the Hr heads in
// head order, then z_adj of this shard's heads -> sb
constexpr int kBtBins = 65536;
constexpr int kBtRow = kBtBins;  // histogram words per row
// monotonic (non-decreasing) value -> bin map of z_adj: equal z, equal bin
__device__ __forceinline__ int bt_bin(double z, double zlo, double scale) {
  const double t = (z - zlo) * scale;
  return t <= 0.0 ? 0 : (t >= (double)(kBtBins - 1) ? kBtBins - 1 : (int)t);
}

template <int kH>
__device__ __forceinline__ void cross_head_store(const SelParams& p, int b, int idx, const double (&zn)[kH],
                                                 int Hr) {
  double mxs = zn[0];
#pragma unroll
  for (int h = 1; h < kH; ++h)
    if (h < Hr) mxs = smax(mxs, zn[h]);
  const bool t_one = (p.temperature == 1.0);
  double e[kH], x[kH];
  double sum = 0.0;
#pragma unroll
  for (int h = 0; h < kH; ++h)
    if (h < Hr) {
      x[h] = t_one ? (zn[h] - mxs) : (zn[h] - mxs) / p.temperature;
      e[h] = exp(x[h]);
      sum += e[h];
    }
  // log(max(e_h / sum, eps)) = x_h - log(sum) unless the responsibility is clipped
  const double ls = log(sum);
  const double le = log(p.eps);
  const double floor_e = p.eps * sum;
#pragma unroll
  for (int h = 0; h < kH; ++h)
    if (h < Hr && h >= p.h_off && h < p.h_off + p.H) {  // this shard's heads only
      const double lr = (e[h] >= floor_e) ? (x[h] - ls) : le;
      const double z = zn[h] + p.alpha_cross * lr;
      const size_t row = (size_t)(b * p.H + h - p.h_off);
      p.sb[row * p.ld + idx] = z;
      if (p.bt_hist)  // one fire-and-forget RED per key (a warp-aggregated match_any version: C3 Selector 186 vs 174 us)
        atomicAdd(&p.bt_hist[row * kBtRow + bt_bin(z, p.bt_zlo, p.bt_scale)], 1u);
    }
}

// ---------------------------------------------------------------------------
// Stage B: soft-NMS per head, then cross-head exclusivity; one thread per
// (b, j), the CTA's 256 positions x H heads (+ halo) staged in shared memory.
template <bool kExp, int kH>
__global__ void __launch_bounds__(kRefineT) sel_refine_kernel(const SelParams p) {
  griddep_wait();
  griddep_launch();
  __shared__ double tile[kH][kRefineT + 2 * kMaxNmsR];
  const int b = blockIdx.y;
  const int j0 = blockIdx.x * kRefineT;
  const Src<kExp> src(p, b);
  const int n = src.n;
  if (j0 >= n) return;
  const int R = p.nms_radius;
  const bool staged = R <= kMaxNmsR;
  // kH = 16 also serves head counts that are not a power of two (runtime guard)
  const int Hr = p.z_all ? p.H_all : (kH == 16 ? p.H : kH);
  // sequence shard: local j covers global J index j + off of ng; the soft-NMS
  // window reaches into the neighbours' edges
  const bool seq = p.edges_all != nullptr;
  const int off = seq ? p.j_off[b] : 0;
  const int ng = seq ? p.n_glob[b] : n;
  if (staged) {
    // every thread stages column t and t + 256 (halo) of all heads; all loads
    // are issued before the first shared store
    const int span = kRefineT + 2 * R;
    const int t0 = threadIdx.x, t1 = threadIdx.x + kRefineT;
    const int ja = j0 - R + t0, jb = j0 - R + t1;
    const bool oka = ja + off >= 0 && ja + off < ng, okb = t1 < span && jb + off < ng;
    const bool loca = ja >= 0 && ja < n, locb = jb < n;
    double va[kH], vb[kH];
#pragma unroll
    for (int h = 0; h < kH; ++h) {
      const double* z = zrow(p, b, h < Hr ? h : 0);
      va[h] = (h < Hr && oka) ? (loca ? z[ja] : halo(p, b * p.H + h, ja + off, R)) : 0.0;
      vb[h] = (h < Hr && okb) ? (locb ? z[jb] : halo(p, b * p.H + h, jb + off, R)) : 0.0;
    }
#pragma unroll
    for (int h = 0; h < kH; ++h) {
      tile[h][t0] = va[h];
      if (t1 < span) tile[h][t1] = vb[h];
    }
    __syncthreads();
  }
  const int idx = j0 + threadIdx.x;
  if (idx >= n) return;
  const int lo = max(-off, idx - R);
  const int hi = min(ng - 1 - off, idx + R);
  double zn[kH];
#pragma unroll
  for (int h = 0; h < kH; ++h) {
    zn[h] = 0.0;
    if (h < Hr) {
      double zj, m;
      if (staged) {
        const double* t = &tile[h][R + threadIdx.x - idx];  // t[j] = z[j] for j in [j0-R, j0+256+R)
        zj = t[idx];
        m = zj;
        for (int i = lo; i <= hi; ++i) m = smax(m, t[i]);
      } else {
        const double* z = zrow(p, b, h);
        zj = z[idx];
        m = zj;
        for (int i = lo; i <= hi; ++i) m = smax(m, z[i]);
      }
      const double gap = m - zj;
      zn[h] = zj - p.alpha_soft * gap;
    }
  }
  cross_head_store<kH>(p, b, idx, zn, Hr);
}

// ---------------------------------------------------------------------------
// Decode Selector, three passes (cache mode, W = 1, alpha = 1, unsharded):
//   sel_pw_kernel   per (request, 512-position chunk, <= 4 heads): the prior's
//                   position factor exp(-beta u^p) (1 - u + eps)^eta once per
//                   position (the same for every head), then per head the chunk
//                   max m_c, p = exp(v - m_c), w = (|k| + eps)^-gamma * factor -> W
//                   (fp64) and the chunk's five sums relative to m_c -> stats.
//   sel_coef_kernel per row: the row max M, the sums rescaled to M (chunk order),
//                   lambda*, a = (1 - lambda) / sum p, b = lambda / sum w.
//   sel_z_kernel    per (request, 256 positions), all heads: p = exp(v - M)
//                   recomputed from the fp32 logits against the ROW max (equal
//                   logits -> equal p, so exact ties are kept), z = log(a p + b w
//                   + eps) for the tile and its soft-NMS halo in shared memory,
//                   soft-NMS, cross-head -> z_adj.
// No P or z_base round trip through HBM.
constexpr int kPwT = 256;
constexpr int kPwPer = 2;
constexpr int kChunk = kPwT * kPwPer;  // positions per statistics chunk
constexpr int kPwHeads = 4;            // heads per CTA (blockIdx.z splits larger groups)

__host__ __device__ __forceinline__ int n_chunks(int n) { return (n + kChunk - 1) / kChunk; }

// kHC: heads per CTA (kPwHeads; 1 for small problems, where 4x the CTAs beat
// sharing the position factor)
// kDef: the default exponents (gamma 1, p 2, eta 0.5) — the same operations
// pow_ref selects at run time (1/x, x*x, sqrt), without the per-element dispatch.
template <int kHT, int kHC = kPwHeads, bool kDef = false>
__global__ void __launch_bounds__(kPwT, 4) sel_pw_kernel(const SelParams p, double* P, double* Wt, double* stats,
                                                      int ld_chunks) {
  griddep_wait();  // PDL: logits come from the preceding dense decode
  griddep_launch();
  if (p.bt_hist) {  // long-row top-k: clear this CTA's share of the histograms sel_z fills next
    const size_t words = (size_t)p.B * p.H * kBtRow / 4;
    const size_t nb = (size_t)gridDim.x * gridDim.y * gridDim.z;
    const size_t cta = ((size_t)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
    const size_t w0 = words * cta / nb, w1 = words * (cta + 1) / nb;
    uint4* h4 = reinterpret_cast<uint4*>(p.bt_hist);
    for (size_t i = w0 + threadIdx.x; i < w1; i += blockDim.x) h4[i] = make_uint4(0u, 0u, 0u, 0u);
  }
  constexpr int kH = kHT < kHC ? kHT : kHC;  // heads of this CTA
  constexpr int kW = kPwT / 32;
  __shared__ double red[kW][kH][5];
  __shared__ double mc[kH];
  const int b = blockIdx.y;
  const int h0 = blockIdx.z * kH;
  const Src<false> src(p, b);
  const int n = src.n;
  const int c0 = blockIdx.x * kChunk;
  if (c0 >= n) return;
  const int Hr = min(kH, (kHT == 16 ? p.H : kHT) - h0);
  if (Hr <= 0) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const double denom_u = src.u_denom();
  double fpos[kPwPer];
  bool bad = false;
#pragma unroll
  for (int i = 0; i < kPwPer; ++i) {
    const int j = c0 + threadIdx.x + i * kPwT;
    if (j < n) {
      const double u = src.u(j, denom_u);
      fpos[i] = kDef ? exp(-p.beta * (u * u)) * sqrt(1.0 - u + p.eps)
                     : exp(-p.beta * pow_ref(u, p.p_curve)) * pow_ref(1.0 - u + p.eps, p.eta);
    } else {
      fpos[i] = 0.0;
    }
  }
  // chunk max per head (starts at kMaskedLogit), finite check
  float v[kH][kPwPer];
#pragma unroll
  for (int h = 0; h < kH; ++h) {
    double m = kMaskedLogit;
#pragma unroll
    for (int i = 0; i < kPwPer; ++i) {
      const int j = c0 + threadIdx.x + i * kPwT;
      const bool ok = h < Hr && j < n;
      v[h][i] = ok ? p.logits32[(size_t)(b * p.H + h0 + h) * p.ld + j] : -INFINITY;
      if (ok) {
        if (!isfinite(v[h][i])) bad = true;
        m = smax(m, (double)v[h][i]);
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = smax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (lane == 0) red[warp][h][0] = m;
  }
  if (bad) raise_error(p.err, SFI_ERR_NON_FINITE_INPUT);
  __syncthreads();
  if (threadIdx.x < Hr) {
    double m = red[0][threadIdx.x][0];
    for (int w = 1; w < kW; ++w) m = smax(m, red[w][threadIdx.x][0]);
    mc[threadIdx.x] = m;
  }
  __syncthreads();
  // p, w, the five sums per head
  bool badn = false;
#pragma unroll
  for (int h = 0; h < kH; ++h) {
    if (h >= Hr) break;
    const int row = b * p.H + h0 + h;
    const double m = mc[h];
    double sp = 0.0, sw = 0.0, spp = 0.0, spw = 0.0, sww = 0.0;
#pragma unroll
    for (int i = 0; i < kPwPer; ++i) {
      const int j = c0 + threadIdx.x + i * kPwT;
      if (j < n) {
        const double vv = (double)v[h][i];
        const double nm = src.norm(row, j);
        if (!isfinite(nm) || nm < 0.0) badn = true;
        const double pj = (vv <= kMaskedLogit) ? 0.0 : exp(vv - m);
        const double wr = (kDef ? 1.0 / (nm + p.eps) : pow_ref(nm + p.eps, -p.gamma)) * fpos[i];
        if (!isfinite(wr) || wr < 0.0) badn = true;
        (void)P;  // p is recomputed by sel_z from the logits (saves its write + read)
        Wt[(size_t)row * p.ld + j] = wr;
        sp += pj;
        sw += wr;
        spp += pj * pj;
        spw += pj * wr;
        sww += wr * wr;
      }
    }
    double x[5] = {sp, sw, spp, spw, sww};
#pragma unroll
    for (int k = 0; k < 5; ++k) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) x[k] += __shfl_xor_sync(0xffffffffu, x[k], o);
      if (lane == 0) red[warp][h][k] = x[k];
    }
  }
  if (badn) raise_error(p.err, SFI_ERR_NON_FINITE_INPUT);
  __syncthreads();
  if (threadIdx.x < Hr * 5) {  // warps in index order: deterministic
    const int h = threadIdx.x / 5, k = threadIdx.x % 5;
    double acc = red[0][h][k];
    for (int w = 1; w < kW; ++w) acc += red[w][h][k];
    double* st = stats + ((size_t)(b * p.H + h0 + h) * ld_chunks + blockIdx.x) * 6;
    st[1 + k] = acc;
    if (k == 0) st[0] = mc[h];
  }
}

// Per row: the row max M and the fused coefficients from the chunk statistics
// (rescaled to M in chunk order): coef[row] = {a = (1 - lambda) / sum p,
// b = lambda / sum w, M}. sel_z forms p = exp(v - M) against the ROW max, as
// row_softmax does (selector.cpp:54-74): equal logits give bit-equal p, so the
// reference's exact ties (equal score -> lower position) survive at any distance.
__global__ void sel_coef_kernel(const SelParams p, const double* __restrict__ stats, double* __restrict__ coef,
                                int ld_chunks) {
  griddep_wait();
  griddep_launch();
  // one warp per row; lanes own chunks c = lane + 32 k; warp-tree reductions (fixed order)
  const int lane = threadIdx.x & 31;
  const int row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (row >= p.B * p.H) return;
  const Src<false> src(p, row / p.H);
  const int n = src.n;
  if (n <= 0) return;
  const double* st = stats + (size_t)row * ld_chunks * 6;
  double* cf = coef + (size_t)row * (ld_chunks + 2);
  const int nc = n_chunks(n);
  double M = kMaskedLogit;
  for (int c = lane; c < nc; c += 32) M = smax(M, st[c * 6]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) M = smax(M, __shfl_xor_sync(0xffffffffu, M, o));
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0, s4 = 0.0;
  for (int c = lane; c < nc; c += 32) {
    const double* x = st + c * 6;
    const double e = exp(x[0] - M);
    s0 += x[1] * e;
    s1 += x[2];
    s2 += x[3] * (e * e);
    s3 += x[4] * e;
    s4 += x[5];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    s0 += __shfl_xor_sync(0xffffffffu, s0, o);
    s1 += __shfl_xor_sync(0xffffffffu, s1, o);
    s2 += __shfl_xor_sync(0xffffffffu, s2, o);
    s3 += __shfl_xor_sync(0xffffffffu, s3, o);
    s4 += __shfl_xor_sync(0xffffffffu, s4, o);
  }
  if (lane == 0 && (s0 <= 0.0 || s1 <= 0.0)) raise_error(p.err, SFI_ERR_EMPTY_SUPPORT);
  // f = p / sum p, r = w / sum w (normalize); fuse (selector.cpp:166-174)
  const double c1 = 1.0 / s0, c2 = 1.0 / s1;
  const double ff = s2 * c1 * c1, fr = s3 * c1 * c2, rr = s4 * c2 * c2;
  const double denom = ff - 2.0 * fr + rr;
  double lambda = 0.0;
  if (fabs(denom) >= p.eps) {
    lambda = (ff - fr) / denom;
    lambda = (lambda < 0.0) ? 0.0 : (p.lambda_clip < lambda) ? p.lambda_clip : lambda;
  }
  if (lane == 0) {
    cf[0] = (1.0 - lambda) * c1;
    cf[1] = lambda * c2;
    cf[2] = M;
  }
}

// The same per row for long rows (C3, C4: 256-512 chunks): one 256-thread CTA per row,
// threads own chunks c = t + 256 k; warp trees then the 8 warps in order (fixed order).
__global__ void __launch_bounds__(256) sel_coef_wide_kernel(const SelParams p, const double* __restrict__ stats,
                                                            double* __restrict__ coef, int ld_chunks) {
  griddep_wait();
  griddep_launch();
  __shared__ double red[8][5];
  __shared__ double sM;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int row = blockIdx.x;
  const Src<false> src(p, row / p.H);
  const int n = src.n;
  if (n <= 0) return;
  const double* st = stats + (size_t)row * ld_chunks * 6;
  double* cf = coef + (size_t)row * (ld_chunks + 2);
  const int nc = n_chunks(n);
  double M = kMaskedLogit;
  for (int c = threadIdx.x; c < nc; c += 256) M = smax(M, st[c * 6]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) M = smax(M, __shfl_xor_sync(0xffffffffu, M, o));
  if (lane == 0) red[warp][0] = M;
  __syncthreads();
  if (threadIdx.x == 0) {
    double m = red[0][0];
    for (int w = 1; w < 8; ++w) m = smax(m, red[w][0]);
    sM = m;
  }
  __syncthreads();
  M = sM;
  double x5[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
  for (int c = threadIdx.x; c < nc; c += 256) {
    const double* x = st + c * 6;
    const double e = exp(x[0] - M);
    x5[0] += x[1] * e;
    x5[1] += x[2];
    x5[2] += x[3] * (e * e);
    x5[3] += x[4] * e;
    x5[4] += x[5];
  }
#pragma unroll
  for (int k = 0; k < 5; ++k) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x5[k] += __shfl_xor_sync(0xffffffffu, x5[k], o);
  }
  __syncthreads();  // red reused
  if (lane == 0)
#pragma unroll
    for (int k = 0; k < 5; ++k) red[warp][k] = x5[k];
  __syncthreads();
  if (threadIdx.x != 0) return;
  double s[5];
#pragma unroll
  for (int k = 0; k < 5; ++k) {
    s[k] = red[0][k];
    for (int w = 1; w < 8; ++w) s[k] += red[w][k];
  }
  if (s[0] <= 0.0 || s[1] <= 0.0) raise_error(p.err, SFI_ERR_EMPTY_SUPPORT);
  const double c1 = 1.0 / s[0], c2 = 1.0 / s[1];
  const double ff = s[2] * c1 * c1, fr = s[3] * c1 * c2, rr = s[4] * c2 * c2;
  const double denom = ff - 2.0 * fr + rr;
  double lambda = 0.0;
  if (fabs(denom) >= p.eps) {
    lambda = (ff - fr) / denom;
    lambda = (lambda < 0.0) ? 0.0 : (p.lambda_clip < lambda) ? p.lambda_clip : lambda;
  }
  cf[0] = (1.0 - lambda) * c1;
  cf[1] = lambda * c2;
  cf[2] = M;
}

template <int kH>
__global__ void __launch_bounds__(kRefineT, kH <= 8 ? 4 : 2) sel_z_kernel(const SelParams p, const double* stats, const double* Wt,
                                                         const double* coef, int ld_chunks) {
  griddep_wait();
  griddep_launch();
  __shared__ double tile[kH][kRefineT + 2 * kMaxNmsR];
  __shared__ double ca[kH];  // (1 - lambda) / sum p
  __shared__ double cm[kH];  // the row max M (p = exp(v - M) is recomputed from the logits, not stored)
  __shared__ double cb[kH];  // lambda / sum w
  const int b = blockIdx.y;
  const int j0 = blockIdx.x * kRefineT;
  const Src<false> src(p, b);
  const int n = src.n;
  if (j0 >= n) return;
  const int R = p.nms_radius;
  const int Hr = kH == 16 ? p.H : kH;
  (void)stats;
  if (threadIdx.x < 3 * Hr) {
    const int h = threadIdx.x / 3, k = threadIdx.x % 3;
    const double v = coef[(size_t)(b * p.H + h) * (ld_chunks + 2) + k];
    if (k == 0) ca[h] = v;
    else if (k == 1) cb[h] = v;
    else cm[h] = v;
  }
  __syncthreads();
  // ---- z_base of the tile and its halo, all heads, into shared memory ----
  const int span = kRefineT + 2 * R;
  for (int it = threadIdx.x; it < span * Hr; it += kRefineT) {
    const int h = it / span, t = it - h * span;
    const int j = j0 - R + t;
    if (j < 0 || j >= n) continue;
    const size_t o = (size_t)(b * p.H + h) * p.ld + j;
    const double v = src.logit(b * p.H + h, 0, j);
    const double pj = (v <= kMaskedLogit) ? 0.0 : exp(v - cm[h]);
    tile[h][t] = log(ca[h] * pj + cb[h] * Wt[o] + p.eps);
  }
  __syncthreads();
  const int idx = j0 + threadIdx.x;
  if (idx >= n) return;
  const int lo = max(0, idx - R);
  const int hi = min(n - 1, idx + R);
  double zn[kH];
#pragma unroll
  for (int h = 0; h < kH; ++h) {
    zn[h] = 0.0;
    if (h < Hr) {
      const double* t = &tile[h][R + threadIdx.x - idx];  // t[j] = z[j] for j in [j0-R, j0+256+R)
      const double zj = t[idx];
      double mm = zj;
      for (int i = lo; i <= hi; ++i) mm = smax(mm, t[i]);
      zn[h] = zj - p.alpha_soft * (mm - zj);
    }
  }
  cross_head_store<kH>(p, b, idx, zn, Hr);
}

// ---------------------------------------------------------------------------
// Stage C: top-k per row.

// Order-preserving key: larger score -> larger key; -0.0 ties +0.0 as in the
// reference comparator (selector.cpp:245 compares with != and >).
__device__ __forceinline__ unsigned long long okey(double x) {
  if (x == 0.0) x = 0.0;
  const unsigned long long u = (unsigned long long)__double_as_longlong(x);
  return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}

// kSmem: the CTA's block of keys lives in dynamic shared memory (one global
// read); otherwise every pass re-reads z from global/L2.
template <bool kExp, bool kSmem, int CS>
__global__ void __launch_bounds__(kT)
    sel_topk_kernel(const SelParams p) {
  griddep_wait();
  griddep_launch();
  extern __shared__ unsigned long long skeys[];
  __shared__ uint32_t hist[2][kBins];
  constexpr int kBPC = kBins / CS;   // bins per CTA
  constexpr int kBPL = kBPC / 32;    // bins per lane in the threshold scan
  __shared__ uint32_t bsum[2][kBPC];
  __shared__ uint32_t slice_tot[2];
  __shared__ int res_tb[2], res_cum[2], res_cnt[2];
  __shared__ unsigned long long cand[kCandCap];       // this CTA's threshold-bucket keys
  __shared__ int ncand;
  __shared__ unsigned long long res_T;
  __shared__ int res_gt;
  __shared__ unsigned long long wbuf[kWarps * 2];
  __shared__ unsigned long long red[2][2];
  __shared__ unsigned long long cta_tot;
  cg::cluster_group cl = cg::this_cluster();
  const int rank = (int)cl.block_rank();
  const int row = blockIdx.y;
  const Src<kExp> src(p, row / p.H);
  const int n = src.n;
  const int K = p.K;
  int32_t* out = p.sel + (size_t)row * K;
  if (n <= 0 || K == 0) {
    if (rank == 0 && threadIdx.x == 0) p.n_sel[row] = 0;
    return;
  }
  if (n <= K) {  // |J| <= k: all of J (selector.cpp:239)
    for (int i = rank * kT + threadIdx.x; i < n; i += CS * kT) out[i] = src.pos(i);
    if (rank == 0 && threadIdx.x == 0) p.n_sel[row] = n;
    return;
  }
  const double* z = p.sb + (size_t)row * p.ld;
  // this CTA's contiguous block of the row
  const int chunk = (n + CS - 1) / CS;
  const int c0 = rank * chunk, c1 = min(n, c0 + chunk);
  const int len = max(0, c1 - c0);
  auto key_at = [&](int i) -> unsigned long long {  // i relative to c0
    return kSmem ? skeys[i] : okey(z[c0 + i]);
  };
  int par = 0;

  // pass 0: stage keys, key range
  unsigned long long mm[2] = {~0ull, ~0ull};  // min key, min ~key (= ~max key)
  for (int i = threadIdx.x; i < len; i += kT) {
    const unsigned long long k = okey(z[c0 + i]);
    if (kSmem) skeys[i] = k;
    mm[0] = k < mm[0] ? k : mm[0];
    mm[1] = ~k < mm[1] ? ~k : mm[1];
  }
  cluster_reduce<2>(mm, 2, wbuf, red, par, cl, OpMinU());  // includes the smem-key barrier
  const unsigned long long kmin = mm[0], kmax = ~mm[1];

  // radix refinement: invariant T in [lo, lo + 2^bits); `above` keys > range.
  // Buffers alternate by pass; 2 cluster barriers per pass.
  unsigned long long lo = kmin;
  int bits = (kmax == kmin) ? 0 : 64 - __clzll((long long)(kmax - kmin));
  int above = 0;
  int pb = 0;
  for (int i = threadIdx.x; i < kBins; i += kT) hist[0][i] = 0;
  __syncthreads();
  while (bits > 0) {
    const int shift = bits > 11 ? bits - 11 : 0;
    const int nb = 1 << (bits - shift);
    uint32_t* hcur = hist[pb];
    for (int i = threadIdx.x; i < len; i += kT) {
      const unsigned long long k = key_at(i);
      if (k >= lo) {
        const unsigned long long d = (k - lo) >> shift;
        if (d < (unsigned long long)nb) atomicAdd(&hcur[d], 1u);
      }
    }
    cl.sync();  // (1) every CTA's histogram complete
    // zero the other buffer for the next pass (its last readers passed barrier (1))
    for (int i = threadIdx.x; i < kBins; i += kT) hist[pb ^ 1][i] = 0;
    uint32_t mine = 0;
    for (int bi = threadIdx.x; bi < kBPC; bi += kT) {
      const int gb = rank * kBPC + bi;
      uint32_t s = 0;
      if (gb < nb)
        for (int r = 0; r < CS; ++r) s += cl.map_shared_rank(hcur, r)[gb];
      bsum[pb][bi] = s;
      mine += s;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, o);
    if ((threadIdx.x & 31) == 0) wbuf[threadIdx.x >> 5] = mine;
    __syncthreads();
    if (threadIdx.x == 0) {
      uint32_t t = 0;
      for (int w = 0; w < kWarps; ++w) t += (uint32_t)wbuf[w];
      slice_tot[pb] = t;
    }
    cl.sync();  // (2) merged slices + their totals published
    // warp 0 of every CTA finds the threshold bucket (same answer cluster-wide):
    // lanes read the 8 slice totals, then the owner slice's 256 bins (8 per
    // lane) over DSMEM in parallel, scanning from the top bin down
    const int need_rem = K - above;
    if (threadIdx.x < 32) {
      const int lane = threadIdx.x;
      const int tr = lane < CS ? (int)*cl.map_shared_rank(&slice_tot[pb], CS - 1 - lane) : 0;
      int inc = tr;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
      }
      const unsigned m1 = __ballot_sync(0xffffffffu, lane < CS && inc >= need_rem);
      const int fl = m1 ? __ffs(m1) - 1 : CS - 1;
      const int own = CS - 1 - fl;
      const int cum = __shfl_sync(0xffffffffu, inc - tr, fl);  // keys in ranks above `own`
      const uint32_t* ob = cl.map_shared_rank(&bsum[pb][0], own);
      uint32_t bv[kBPL];
      int lsum = 0;
#pragma unroll
      for (int k = 0; k < kBPL; ++k) {
        bv[k] = ob[kBPC - 1 - (lane * kBPL + k)];  // descending bins
        lsum += (int)bv[k];
      }
      int inc2 = lsum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, inc2, o);
        if (lane >= o) inc2 += y;
      }
      const unsigned m2 = __ballot_sync(0xffffffffu, cum + inc2 >= need_rem);
      const int fl2 = m2 ? __ffs(m2) - 1 : 31;
      if (lane == fl2) {
        int c2 = cum + inc2 - lsum;
        int tb = own * kBPC + (kBPC - 1 - lane * kBPL - (kBPL - 1));
        int cnt = 0;
#pragma unroll
        for (int k = 0; k < kBPL; ++k) {
          if (c2 + (int)bv[k] >= need_rem) {
            tb = own * kBPC + (kBPC - 1 - (lane * kBPL + k));
            cnt = (int)bv[k];
            break;
          }
          c2 += (int)bv[k];
        }
        res_tb[pb] = tb;
        res_cum[pb] = c2;
        res_cnt[pb] = cnt;
      }
    }
    __syncthreads();
    const int tb = res_tb[pb];
    above += res_cum[pb];  // keys in buckets above tb are above the threshold
    lo += (unsigned long long)tb << shift;
    bits = shift;
    pb ^= 1;
    if (bits > 0 && res_cnt[pb ^ 1] <= kCandCap) {
      // Candidate shortcut: the threshold bucket [lo, lo + 2^bits) holds few
      // keys; gather them and rank them directly instead of more radix passes.
      if (threadIdx.x == 0) ncand = 0;
      __syncthreads();
      for (int i = threadIdx.x; i < len; i += kT) {
        const unsigned long long k = key_at(i);
        if (k >= lo && ((k - lo) >> bits) == 0ull) cand[atomicAdd(&ncand, 1)] = k;
      }
      cl.sync();  // every CTA's candidates complete
      if (rank == 0) {
        // gather all candidates (total <= kCandCap) into call[], CTA order; call
        // aliases the histogram buffer of the pass just finished (no reader left)
        unsigned long long* call = reinterpret_cast<unsigned long long*>(hist[pb ^ 1]);
        int off = 0;
        for (int r = 0; r < CS; ++r) {
          const int nr = *cl.map_shared_rank(&ncand, r);
          const unsigned long long* src = cl.map_shared_rank(cand, r);
          for (int i = threadIdx.x; i < nr; i += kT) call[off + i] = src[i];
          off += nr;
        }
        __syncthreads();
        // T = the need-th largest: #(> T) < need <= #(>= T)
        const int need_rem2 = K - above;
        for (int i = threadIdx.x; i < off; i += kT) {
          const unsigned long long v = call[i];
          int gt = 0, ge = 0;
          for (int j = 0; j < off; ++j) {
            gt += call[j] > v;
            ge += call[j] >= v;
          }
          if (gt < need_rem2 && ge >= need_rem2) {  // same (T, gt) for all ties
            res_T = v;
            res_gt = gt;
          }
        }
      }
      cl.sync();  // rank 0's answer published
      lo = *cl.map_shared_rank(&res_T, 0);
      above += *cl.map_shared_rank(&res_gt, 0);
      bits = 0;
    }
  }
  const unsigned long long T = lo;
  const int need = K - above;

  // ordered emission: blocked sub-ranges, packed (gt, eq) exclusive scan
  const int E = (len + kT - 1) / kT;
  const int e0 = threadIdx.x * E, e1 = min(len, e0 + E);
  unsigned long long cnt = 0;
  for (int i = e0; i < e1; ++i) {
    const unsigned long long k = key_at(i);
    if (k > T) cnt += (1ull << 32);
    else if (k == T) cnt += 1ull;
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned long long inc = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  __syncthreads();  // wbuf reuse
  if (lane == 31) wbuf[warp] = inc;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long run = 0;
    for (int w = 0; w < kWarps; ++w) {
      const unsigned long long t = wbuf[w];
      wbuf[w] = run;
      run += t;
    }
    cta_tot = run;
  }
  cl.sync();
  unsigned long long base = wbuf[warp] + (inc - cnt);
  for (int r = 0; r < rank; ++r) base += *cl.map_shared_rank(&cta_tot, r);
  int gt_b = (int)(base >> 32), eq_b = (int)(base & 0xffffffffu);
  for (int i = e0; i < e1; ++i) {
    const unsigned long long k = key_at(i);
    if (k > T) {
      out[gt_b + min(eq_b, need)] = src.pos(c0 + i);
      ++gt_b;
    } else if (k == T) {
      if (eq_b < need) out[gt_b + eq_b] = src.pos(c0 + i);
      ++eq_b;
    }
  }
  if (rank == 0 && threadIdx.x == 0) p.n_sel[row] = K;
  cl.sync();
}

// Single-CTA top-k for rows of up to kTopkCtaMax positions: no cluster
// barriers. The high 32 bits of every order-preserving key live in shared
// memory; radix passes (11-bit digits) and the candidate ranking run on them,
// and the full 64-bit key is read back only for elements that tie with the
// threshold on the high word. Same output contract as sel_topk_kernel.
constexpr int kTopkCtaT = 1024;
constexpr int kTopkCtaMax = kTopkCtaMaxPositions;

template <bool kExp>
__global__ void __launch_bounds__(kTopkCtaT) sel_topk_cta_kernel(const SelParams p) {
  griddep_wait();
  griddep_launch();
  extern __shared__ uint32_t shi[];              // [n] high words
  __shared__ uint32_t hist[kBins];
  __shared__ unsigned long long cand[kCandCap];  // full keys of threshold-bucket elements
  __shared__ uint32_t wred[32][2];
  __shared__ int s_ncand, s_tb, s_cum, s_cnt, s_gt;
  __shared__ unsigned long long s_T;
  __shared__ unsigned long long wtot[32];
  constexpr int kW = kTopkCtaT / 32;
  const int row = blockIdx.x;
  const Src<kExp> src(p, row / p.H);
  const int n = src.n;
  const int K = p.K;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int32_t* out = p.sel + (size_t)row * K;
  if (n <= 0 || K == 0) {
    if (threadIdx.x == 0) p.n_sel[row] = 0;
    return;
  }
  if (n <= K) {
    for (int i = threadIdx.x; i < n; i += kTopkCtaT) out[i] = src.pos(i);
    if (threadIdx.x == 0) p.n_sel[row] = n;
    return;
  }
  const double* z = p.sb + (size_t)row * p.ld;
  // pass 0: high words into smem + their range
  uint32_t hmin = 0xffffffffu, hmax = 0u;
  constexpr int kLU = 8;  // loads in flight per thread
  for (int i0 = threadIdx.x; i0 < n; i0 += kLU * kTopkCtaT) {
    double zv[kLU];
#pragma unroll
    for (int u = 0; u < kLU; ++u) {
      const int i = i0 + u * kTopkCtaT;
      zv[u] = i < n ? z[i] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < kLU; ++u) {
      const int i = i0 + u * kTopkCtaT;
      if (i < n) {
        const uint32_t h = (uint32_t)(okey(zv[u]) >> 32);
        shi[i] = h;
        hmin = min(hmin, h);
        hmax = max(hmax, h);
      }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    hmin = min(hmin, __shfl_xor_sync(0xffffffffu, hmin, o));
    hmax = max(hmax, __shfl_xor_sync(0xffffffffu, hmax, o));
  }
  if (lane == 0) {
    wred[warp][0] = hmin;
    wred[warp][1] = hmax;
  }
  __syncthreads();
  hmin = wred[0][0];
  hmax = wred[0][1];
  for (int w = 1; w < kW; ++w) {
    hmin = min(hmin, wred[w][0]);
    hmax = max(hmax, wred[w][1]);
  }
  // radix over the high word: invariant threshold high word in [lo, lo + 2^bits)
  uint32_t lo = hmin;
  int bits = (hmax == hmin) ? 0 : 32 - __clz((int)(hmax - hmin));
  int above = 0;
  bool resolved = false;
  unsigned long long T = 0;
  // keys with high word in the current range: all n at first, then the count of
  // the digit bucket each radix pass narrows the range to
  int cnt_range = n;
  while (true) {
    // candidate shortcut (also the exit once the high word is pinned)
    if (cnt_range <= kCandCap) {
      if (threadIdx.x == 0) s_ncand = 0;
      __syncthreads();
      for (int i = threadIdx.x; i < n; i += kTopkCtaT) {
        const uint32_t h = shi[i];
        if (h >= lo && (bits >= 32 || ((h - lo) >> bits) == 0u)) cand[atomicAdd(&s_ncand, 1)] = okey(z[i]);
      }
      __syncthreads();
      const int nc = s_ncand;
      const int need_rem = K - above;
      for (int i = threadIdx.x; i < nc; i += kTopkCtaT) {
        const unsigned long long v = cand[i];
        int gt = 0, ge = 0;
        for (int j = 0; j < nc; ++j) {
          gt += cand[j] > v;
          ge += cand[j] >= v;
        }
        if (gt < need_rem && ge >= need_rem) {
          s_T = v;
          s_gt = gt;
        }
      }
      __syncthreads();
      T = s_T;
      above += s_gt;
      resolved = true;
      break;
    }
    if (bits == 0) break;  // > kCandCap keys share one high word: exact pass below
    const int shift = bits > 11 ? bits - 11 : 0;
    const int nb = 1 << (bits - shift);
    for (int i = threadIdx.x; i < kBins; i += kTopkCtaT) hist[i] = 0;
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += kTopkCtaT) {
      const uint32_t h = shi[i];
      if (h >= lo) {
        const uint32_t d = (h - lo) >> shift;
        if (d < (uint32_t)nb) atomicAdd(&hist[d], 1u);
      }
    }
    __syncthreads();
    if (warp == 0) {  // threshold bucket, scanning from the top bin down (64 bins per lane)
      const int need_rem = K - above;
      int lsum = 0;
      for (int k = 0; k < kBins / 32; ++k) lsum += (int)hist[kBins - 1 - (lane * (kBins / 32) + k)];
      int inc = lsum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
      }
      const unsigned m = __ballot_sync(0xffffffffu, inc >= need_rem);
      const int fl = m ? __ffs(m) - 1 : 31;
      if (lane == fl) {
        int c2 = inc - lsum, tb = 0, cnt = 0;
        for (int k = 0; k < kBins / 32; ++k) {
          const int bi = kBins - 1 - (lane * (kBins / 32) + k);
          const int c = (int)hist[bi];
          if (c2 + c >= need_rem) {
            tb = bi;
            cnt = c;
            break;
          }
          c2 += c;
        }
        s_tb = tb;
        s_cum = c2;
        s_cnt = cnt;
      }
    }
    __syncthreads();
    above += s_cum;
    lo += (uint32_t)s_tb << shift;
    bits = shift;
    cnt_range = s_cnt;
    __syncthreads();
  }
  if (!resolved) {
    // Rare: more than kCandCap keys share the threshold high word `lo`.
    // Resolve the low word by radix passes over those elements (global reads).
    uint32_t llo = 0;
    int lbits = 32;
    while (lbits > 0) {
      const int shift = lbits > 11 ? lbits - 11 : 0;
      const int nb = 1 << (lbits - shift);
      for (int i = threadIdx.x; i < kBins; i += kTopkCtaT) hist[i] = 0;
      __syncthreads();
      for (int i = threadIdx.x; i < n; i += kTopkCtaT) {
        if (shi[i] != lo) continue;
        const uint32_t l = (uint32_t)okey(z[i]);
        if (l >= llo) {
          const uint32_t d = (l - llo) >> shift;
          if (d < (uint32_t)nb) atomicAdd(&hist[d], 1u);
        }
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        const int need_rem = K - above;
        int c2 = 0, tb = 0;
        for (int bi = nb - 1; bi >= 0; --bi) {
          if (c2 + (int)hist[bi] >= need_rem) {
            tb = bi;
            break;
          }
          c2 += (int)hist[bi];
        }
        s_tb = tb;
        s_cum = c2;
      }
      __syncthreads();
      above += s_cum;
      llo += (uint32_t)s_tb << shift;
      lbits = shift;
      __syncthreads();
    }
    T = ((unsigned long long)lo << 32) | llo;
  }
  const int need = K - above;
  const uint32_t Th = (uint32_t)(T >> 32);

  // ordered emission: blocked ranges, packed (gt, eq) exclusive scan
  const int E = (n + kTopkCtaT - 1) / kTopkCtaT;
  const int e0 = threadIdx.x * E, e1 = min(n, e0 + E);
  auto cls = [&](int i) -> int {  // 2: > T, 1: == T, 0: < T
    const uint32_t h = shi[i];
    if (h != Th) return h > Th ? 2 : 0;
    const unsigned long long k = okey(z[i]);
    return k > T ? 2 : (k == T ? 1 : 0);
  };
  // classify this thread's E (<= 48) elements once; reads are rotated by the
  // thread index so a warp's 32 threads hit 32 different banks
  const int len = max(0, e1 - e0);
  unsigned long long gtm = 0, eqm = 0;  // bit k: element e0 + k
  {
    const int rot = len ? (int)(threadIdx.x % (unsigned)len) : 0;
    for (int kk = 0; kk < len; ++kk) {
      int k = kk + rot;
      if (k >= len) k -= len;
      const int c = cls(e0 + k);
      if (c == 2) gtm |= 1ull << k;
      else if (c == 1) eqm |= 1ull << k;
    }
  }
  const unsigned long long cnt = ((unsigned long long)__popcll(gtm) << 32) | (unsigned long long)__popcll(eqm);
  unsigned long long inc = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) wtot[warp] = inc;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long run = 0;
    for (int w = 0; w < kW; ++w) {
      const unsigned long long t = wtot[w];
      wtot[w] = run;
      run += t;
    }
  }
  __syncthreads();
  const unsigned long long base = wtot[warp] + (inc - cnt);
  int gt_b = (int)(base >> 32), eq_b = (int)(base & 0xffffffffu);
  unsigned long long sel = gtm | eqm;
  while (sel) {  // position order within the block
    const int k = __ffsll((long long)sel) - 1;
    sel &= sel - 1;
    if ((gtm >> k) & 1ull) {
      out[gt_b + min(eq_b, need)] = src.pos(e0 + k);
      ++gt_b;
    } else {
      if (eq_b < need) out[gt_b + eq_b] = src.pos(e0 + k);
      ++eq_b;
    }
  }
  if (threadIdx.x == 0) p.n_sel[row] = K;
}

void fill_cfg(SelParams& p, const sfi_selector_params& prm) {
  p.alpha = prm.alpha;
  p.gamma = prm.gamma;
  p.beta = prm.beta;
  p.p_curve = prm.p_curve;
  p.eta = prm.eta;
  p.lambda_clip = prm.lambda_clip;
  p.alpha_soft = prm.alpha_soft;
  p.alpha_cross = prm.alpha_cross;
  p.temperature = prm.temperature;
  p.eps = prm.epsilon;
  p.nms_radius = prm.nms_radius;
}

template <void (*Fn)(SelParams)>
cudaError_t launch_topk_cluster(dim3 grid, size_t smem, int cs, cudaStream_t st, const SelParams& p) {
  cudaError_t e = ensure_kernel_attrs(reinterpret_cast<const void*>(Fn),
                                      kTopkSmemKeys * (int)sizeof(unsigned long long));
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(kT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cs;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  return cudaLaunchKernelEx(&cfg, Fn, p);
}

template <bool kExp>
cudaError_t launch_topk(const SelParams& p, int rows, int n_max, cudaStream_t st) {
  // SFI_TOPK_CLUSTER=1: 8-CTA cluster top-k for every row length; =4: 4-CTA clusters
  static const int force_cluster = [] {
    const char* e = std::getenv("SFI_TOPK_CLUSTER");
    return e ? std::atoi(e) : 0;
  }();
  if (n_max <= kTopkCtaMax && !force_cluster) {
    const size_t smem = (size_t)std::max(n_max, 1) * sizeof(uint32_t);
    cudaError_t e = ensure_kernel_attrs(reinterpret_cast<const void*>(sel_topk_cta_kernel<kExp>),
                                        kTopkCtaMax * (int)sizeof(uint32_t));
    if (e != cudaSuccess) return e;
    return launch_k(sel_topk_cta_kernel<kExp>, dim3(rows), dim3(kTopkCtaT), smem, st, p);
  }
  const int cs = (force_cluster == 4) ? 4 : kCS;
  const int chunk = (n_max + cs - 1) / cs;
  const dim3 gc(cs, (unsigned)rows);
  if (chunk <= kTopkSmemKeys) {
    const size_t smem = (size_t)std::max(chunk, 1) * sizeof(unsigned long long);
    return cs == 4 ? launch_topk_cluster<sel_topk_kernel<kExp, true, 4>>(gc, smem, 4, st, p)
                   : launch_topk_cluster<sel_topk_kernel<kExp, true, kCS>>(gc, smem, kCS, st, p);
  }
  return cs == 4 ? launch_topk_cluster<sel_topk_kernel<kExp, false, 4>>(gc, 0, 4, st, p)
                 : launch_topk_cluster<sel_topk_kernel<kExp, false, kCS>>(gc, 0, kCS, st, p);
}

// ---------------------------------------------------------------------------
// Top-k of long rows (|J| > kTopkCtaMax: C3 131K, C4 262K), rows x segments
// wide instead of one 8-CTA cluster per row. sel_z has added every z_adj to a
// per-row histogram of kBtBins value bins over [zlo, zhi], the bounds z_adj
// can take (z_base in [log eps, log(1 + eps)], lowered by at most
// (alpha_soft + alpha_cross) |log eps|); the bin map is monotonic, so
//   sel_bt_thresh  (8-CTA cluster  the bin b* holding the K-th largest key; keys in
//                   per row)       higher bins are selected
//   sel_bt_scan    (segment, row)  per segment: count of keys above b*; keys in b* listed;
//                                  the last segment CTA of a row to arrive then picks the
//                                  exact threshold (key, index) among the listed keys
//                                  (bitonic sort in shared memory, radix select beyond)
//                                  and each segment's output offset
//   sel_bt_emit    (segment, row)  the selected positions, ascending
// Same output contract as sel_topk_kernel (score desc, position asc; ties by position).
constexpr int kBtSmemCand = 2048;
constexpr int kBtMeta = 16;  // row state words
constexpr int kBtMaxSeg = 64;

struct BtBuf {
  uint32_t* hist;  // [rows][kBtBins]
  int32_t* cand;   // [rows][Lmax] listed indices
  int32_t* meta;   // [rows][kBtMeta]: b*, above, need, listed, Tk hi, Tk lo, Ti, mode (1: n <= K / empty),
                   //   scan arrivals
  int32_t* seg;    // [rows][kBtMaxSeg][2]: count above b*, output offset
  int P;           // segments per row
};

__host__ __device__ __forceinline__ int bt_seg_start(int s, int n, int P) { return (int)(((long long)s * n) / P); }

template <int kT, typename T>
__device__ __forceinline__ T block_excl_scan(T v, T* wsum, T& total) {
  constexpr int kW = kT / 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  T inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const T y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) wsum[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    T w = lane < kW ? wsum[lane] : T(0);
    T wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const T y = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += y;
    }
    if (lane < kW) wsum[lane] = wi - w;
    if (lane == kW - 1) wsum[kW] = wi;
  }
  __syncthreads();
  total = wsum[kW];
  const T r = wsum[warp] + inc - v;
  __syncthreads();
  return r;
}

constexpr int kBtThCS = 8;                      // thresh: CTAs per row (one cluster)
constexpr int kBtThT = 256;
constexpr int kBtChunks = kBtBins / 64;         // 64-bin chunks per row
constexpr int kBtThChunks = kBtChunks / kBtThCS;  // chunks per CTA

// The bin b* holding the K-th largest key of a row: one 8-CTA cluster per row.
// Chunk c = bins [kBtBins - 64 (c + 1), kBtBins - 64 c) (descending); CTA r sums
// chunks [r kBtThChunks, (r + 1) kBtThChunks) with coalesced 256-byte reads (16
// per warp in flight), rank 0 scans all chunk sums over DSMEM, then resolves the
// 64 bins of the chunk holding the K-th key.
__global__ void __cluster_dims__(kBtThCS, 1, 1) __launch_bounds__(kBtThT)
    sel_bt_thresh_kernel(const SelParams p, const BtBuf bt) {
  griddep_wait();
  griddep_launch();
  __shared__ uint32_t csum[kBtThChunks];
  __shared__ uint32_t wsum[33];
  __shared__ int s_c;
  __shared__ uint32_t s_before;
  cg::cluster_group cl = cg::this_cluster();
  const int rank = (int)cl.block_rank();
  const int row = blockIdx.y;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const Src<false> src(p, row / p.H);
  const int n = src.n, K = p.K;
  int32_t* m = bt.meta + (size_t)row * kBtMeta;
  const uint32_t* h = bt.hist + (size_t)row * kBtRow;
  const bool active = n > K && K > 0;
  constexpr int kPerWarp = kBtThChunks / (kBtThT / 32);
  static_assert(kPerWarp == 16, "16 chunk reads in flight per lane");
  if (active) {
    uint2 v[kPerWarp];
    const int c0 = rank * kBtThChunks + warp * kPerWarp;
#pragma unroll
    for (int k = 0; k < kPerWarp; ++k) v[k] = __ldcg(reinterpret_cast<const uint2*>(h + kBtBins - 64 * (c0 + k + 1)) + lane);
#pragma unroll
    for (int k = 0; k < kPerWarp; ++k) {
      uint32_t x = v[k].x + v[k].y;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
      if (lane == k) csum[warp * kPerWarp + k] = x;
    }
  }
  cl.sync();  // every CTA's chunk sums visible cluster-wide
  if (rank == 0 && active) {
    // thread t owns chunks 4t .. 4t + 3 (kBtChunks = 4 x kBtThT), read over DSMEM
    static_assert(kBtChunks == 4 * kBtThT, "four chunk sums per thread");
    const int c0 = 4 * threadIdx.x;
    const uint32_t* rs = cl.map_shared_rank(csum, c0 / kBtThChunks);
    uint32_t a[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) a[k] = rs[(c0 % kBtThChunks) + k];
    const uint32_t mine = a[0] + a[1] + a[2] + a[3];
    uint32_t total;
    uint32_t before = block_excl_scan<kBtThT>(mine, wsum, total);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (before < (uint32_t)K && before + a[k] >= (uint32_t)K) {
        s_c = c0 + k;
        s_before = before;
      }
      before += a[k];
    }
  }
  cl.sync();  // rank 0 done reading the peers' sums
  if (rank != 0) return;
  if (active && warp == 0) {  // the 64 bins of chunk s_c, descending: lane pairs, warp prefix
    const int c = s_c;
    const int top = kBtBins - 64 * c;  // bins [top - 64, top)
    const uint32_t v1 = __ldcg(h + top - 1 - 2 * lane), v2 = __ldcg(h + top - 2 - 2 * lane);
    uint32_t inc = v1 + v2;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += y;
    }
    const uint32_t ex = s_before + inc - v1 - v2;  // keys in bins above this lane's pair
    const bool hit1 = ex < (uint32_t)K && ex + v1 >= (uint32_t)K;
    const bool hit2 = !hit1 && ex + v1 < (uint32_t)K && ex + v1 + v2 >= (uint32_t)K;
    if (hit1) {
      m[0] = top - 1 - 2 * lane;
      m[1] = (int32_t)ex;
      m[2] = K - (int32_t)ex;
    } else if (hit2) {
      m[0] = top - 2 - 2 * lane;
      m[1] = (int32_t)(ex + v1);
      m[2] = K - (int32_t)(ex + v1);
    }
  }
  if (threadIdx.x == 0) {
    m[3] = 0;
    m[7] = active ? 0 : 1;
    m[8] = 0;  // scan arrivals (also reset by the picking CTA; here in case a call was cut short)
  }
  // the histograms are cleared by sel_pw at the start of every Selector call
}

constexpr int kBtScanT = 256;

template <int kT>
__device__ __forceinline__ void bt_pick_row(const SelParams& p, const BtBuf& bt, int row);

__global__ void __launch_bounds__(kBtScanT) sel_bt_scan_kernel(const SelParams p, const BtBuf bt) {
  griddep_wait();
  griddep_launch();
  __shared__ uint32_t wsum[33];
  const int seg = blockIdx.x, row = blockIdx.y;
  int32_t* m = bt.meta + (size_t)row * kBtMeta;
  if (m[7]) return;
  const Src<false> src(p, row / p.H);
  const int n = src.n;
  const int s0 = bt_seg_start(seg, n, bt.P), s1 = bt_seg_start(seg + 1, n, bt.P);
  const int bstar = m[0];
  const double* z = p.sb + (size_t)row * p.ld;
  int32_t* cand = bt.cand + (size_t)row * p.Lmax;
  uint32_t cnt = 0;
  for (int i0 = s0 + threadIdx.x; i0 < s1; i0 += 4 * kBtScanT) {
    double zv[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) zv[u] = (i0 + u * kBtScanT < s1) ? z[i0 + u * kBtScanT] : 0.0;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int i = i0 + u * kBtScanT;
      if (i >= s1) break;
      const int bn = bt_bin(zv[u], p.bt_zlo, p.bt_scale);
      if (bn > bstar) ++cnt;
      else if (bn == bstar) cand[atomicAdd(&m[3], 1)] = i;
    }
  }
  uint32_t total;
  block_excl_scan<kBtScanT>(cnt, wsum, total);
  __shared__ int s_last;
  if (threadIdx.x == 0) bt.seg[((size_t)row * kBtMaxSeg + seg) * 2] = (int32_t)total;
  __threadfence();  // every thread: its listed keys (thread 0: the count) before the arrival
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(&m[8], 1) == bt.P - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();  // every segment's count and listed keys are visible
  bt_pick_row<kBtScanT>(p, bt, row);
  if (threadIdx.x == 0) m[8] = 0;  // arrivals reset for the next call
}

// (key desc, index asc) ordering of listed elements
__device__ __forceinline__ bool bt_before(unsigned long long ka, int ia, unsigned long long kb, int ib) {
  return ka > kb || (ka == kb && ia < ib);
}

// The exact threshold (key, index) among a row's listed keys and every segment's
// output offset; run by the last scan CTA of the row to arrive (kT threads).
template <int kT>
__device__ __forceinline__ void bt_pick_row(const SelParams& p, const BtBuf& bt, int row) {
  __shared__ unsigned long long sk[kBtSmemCand];
  __shared__ int si[kBtSmemCand];
  __shared__ uint32_t hist[256];
  __shared__ int segcnt[kBtMaxSeg];
  __shared__ unsigned long long s_tk;
  __shared__ int s_ti, s_gt;
  int32_t* m = bt.meta + (size_t)row * kBtMeta;
  const Src<false> src(p, row / p.H);
  const int n = src.n;
  const int listed = __ldcg(&m[3]), need = m[2];
  const double* z = p.sb + (size_t)row * p.ld;
  const int32_t* cand = bt.cand + (size_t)row * p.Lmax;
  if (threadIdx.x < kBtMaxSeg) segcnt[threadIdx.x] = 0;
  if (listed <= kBtSmemCand) {
    // bitonic sort of the listed (key, index) pairs, padded to a power of two
    int np2 = 1;
    while (np2 < listed) np2 <<= 1;
    for (int i = threadIdx.x; i < np2; i += kT) {
      if (i < listed) {
        sk[i] = okey(__ldcg(&z[__ldcg(&cand[i])]));
        si[i] = __ldcg(&cand[i]);
      } else {
        sk[i] = 0ull;
        si[i] = 0x7fffffff;
      }
    }
    __syncthreads();
    for (int k = 2; k <= np2; k <<= 1)
      for (int j = k >> 1; j > 0; j >>= 1) {
        for (int i = threadIdx.x; i < np2; i += kT) {
          const int ij = i ^ j;
          if (ij > i) {
            const bool up = (i & k) == 0;  // this run sorted "before" first
            const bool swap = up ? bt_before(sk[ij], si[ij], sk[i], si[i]) : bt_before(sk[i], si[i], sk[ij], si[ij]);
            if (swap) {
              const unsigned long long tk = sk[i];
              sk[i] = sk[ij];
              sk[ij] = tk;
              const int ti = si[i];
              si[i] = si[ij];
              si[ij] = ti;
            }
          }
        }
        __syncthreads();
      }
    if (threadIdx.x == 0) {
      s_tk = sk[need - 1];
      s_ti = si[need - 1];
    }
  } else {
    // radix select over the listed keys in global memory: the need-th largest key
    // Tk (8-bit digits), then the (need - #(> Tk))-th smallest index among key == Tk
    unsigned long long prefix = 0ull, pmask = 0ull;
    int rem = need;
    for (int shift = 56; shift >= 0; shift -= 8) {
      for (int i = threadIdx.x; i < 256; i += kT) hist[i] = 0u;
      __syncthreads();
      for (int i = threadIdx.x; i < listed; i += kT) {
        const unsigned long long k = okey(__ldcg(&z[__ldcg(&cand[i])]));
        if ((k & pmask) == prefix) atomicAdd(&hist[(k >> shift) & 255], 1u);
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        int c = 0, d = 255;
        for (; d > 0; --d) {
          if (c + (int)hist[d] >= rem) break;
          c += (int)hist[d];
        }
        s_gt = c;
        s_tk = (unsigned long long)d;
      }
      __syncthreads();
      rem -= s_gt;
      prefix |= s_tk << shift;
      pmask |= 255ull << shift;
      __syncthreads();
    }
    // index among the rem-th smallest with key == prefix
    uint32_t iprefix = 0u, imask = 0u;
    for (int shift = 24; shift >= 0; shift -= 8) {
      for (int i = threadIdx.x; i < 256; i += kT) hist[i] = 0u;
      __syncthreads();
      for (int i = threadIdx.x; i < listed; i += kT) {
        const int ix = __ldcg(&cand[i]);
        if (okey(__ldcg(&z[ix])) == prefix && ((uint32_t)ix & imask) == iprefix) atomicAdd(&hist[((uint32_t)ix >> shift) & 255], 1u);
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        int c = 0, d = 0;
        for (; d < 255; ++d) {
          if (c + (int)hist[d] >= rem) break;
          c += (int)hist[d];
        }
        s_gt = c;
        s_ti = d;
      }
      __syncthreads();
      rem -= s_gt;
      iprefix |= (uint32_t)s_ti << shift;
      imask |= 255u << shift;
      __syncthreads();
    }
    if (threadIdx.x == 0) {
      s_tk = prefix;
      s_ti = (int)iprefix;
    }
  }
  __syncthreads();
  const unsigned long long Tk = s_tk;
  const int Ti = s_ti;
  // selected listed elements per segment
  for (int i = threadIdx.x; i < listed; i += kT) {
    const int ix = __ldcg(&cand[i]);
    const unsigned long long k = okey(__ldcg(&z[ix]));
    if (!bt_before(Tk, Ti, k, ix)) {  // (k, ix) at or before the threshold element
      int sgi = (int)(((long long)ix * bt.P) / n);
      while (sgi + 1 < bt.P && bt_seg_start(sgi + 1, n, bt.P) <= ix) ++sgi;
      while (sgi > 0 && bt_seg_start(sgi, n, bt.P) > ix) --sgi;
      atomicAdd(&segcnt[sgi], 1);
    }
  }
  __syncthreads();
  static_assert(kBtMaxSeg == 64, "two lanes' segments per thread of warp 0");
  if (threadIdx.x < 32) {  // segment output offsets: exclusive prefix of (above b*) + (selected listed)
    int32_t* e = bt.seg + (size_t)row * kBtMaxSeg * 2;
    const int s0 = 2 * threadIdx.x, s1 = s0 + 1;
    const int c0 = s0 < bt.P ? __ldcg(&e[2 * s0]) + segcnt[s0] : 0;
    const int c1 = s1 < bt.P ? __ldcg(&e[2 * s1]) + segcnt[s1] : 0;
    int inc = c0 + c1;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, inc, o);
      if ((int)threadIdx.x >= o) inc += y;
    }
    const int ex = inc - c0 - c1;
    if (s0 < bt.P) e[2 * s0 + 1] = ex;
    if (s1 < bt.P) e[2 * s1 + 1] = ex + c0;
    if (threadIdx.x == 0) {
      m[4] = (int32_t)(Tk >> 32);
      m[5] = (int32_t)(Tk & 0xffffffffull);
      m[6] = Ti;
    }
  }
}

constexpr int kBtEmitTiles = 32;  // 256-key tiles per segment held in registers (flags)

__global__ void __launch_bounds__(kBtScanT) sel_bt_emit_kernel(const SelParams p, const BtBuf bt) {
  griddep_wait();
  griddep_launch();
  constexpr int kW = kBtScanT / 32;
  __shared__ int wcnt[kBtEmitTiles * kW + 1];
  const int seg = blockIdx.x, row = blockIdx.y;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int32_t* m = bt.meta + (size_t)row * kBtMeta;
  const Src<false> src(p, row / p.H);
  const int n = src.n, K = p.K;
  int32_t* out = p.sel + (size_t)row * K;
  const int s0 = bt_seg_start(seg, n, bt.P), s1 = bt_seg_start(seg + 1, n, bt.P);
  if (m[7]) {  // empty J, K = 0, or |J| <= K: all of J (selector.cpp:238-239)
    if (n > 0 && K > 0)
      for (int i = s0 + threadIdx.x; i < s1; i += kBtScanT) out[i] = src.pos(i);
    if (seg == 0 && threadIdx.x == 0) p.n_sel[row] = (n > 0 && K > 0) ? n : 0;
    return;
  }
  const int bstar = m[0];
  const unsigned long long Tk = ((unsigned long long)(uint32_t)m[4] << 32) | (uint32_t)m[5];
  const int Ti = m[6];
  const double* z = p.sb + (size_t)row * p.ld;
  int o_base = bt.seg[((size_t)row * kBtMaxSeg + seg) * 2 + 1];
  // rounds of up to kBtEmitTiles tiles: flags in a register bitmask, counts per (tile, warp)
  for (int r0 = s0; r0 < s1; r0 += kBtEmitTiles * kBtScanT) {
    double zv[kBtEmitTiles];
#pragma unroll
    for (int u = 0; u < kBtEmitTiles; ++u) {
      const int i = r0 + u * kBtScanT + threadIdx.x;
      zv[u] = i < s1 ? z[i] : 0.0;
    }
    uint32_t flags = 0u;
#pragma unroll
    for (int u = 0; u < kBtEmitTiles; ++u) {
      const int i = r0 + u * kBtScanT + threadIdx.x;
      bool f = false;
      if (i < s1) {
        const int bn = bt_bin(zv[u], p.bt_zlo, p.bt_scale);
        f = bn != bstar ? bn > bstar : !bt_before(Tk, Ti, okey(zv[u]), i);
      }
      const unsigned bal = __ballot_sync(0xffffffffu, f);
      if (lane == 0) wcnt[u * kW + warp] = __popc(bal);
      flags |= (f ? 1u : 0u) << u;
    }
    __syncthreads();
    if (warp == 0) {  // exclusive prefix over (tile, warp) in position order
      int carry = 0;
      for (int b0 = 0; b0 < kBtEmitTiles * kW; b0 += 32) {
        const int v = wcnt[b0 + lane];
        int inc = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, inc, o);
          if (lane >= o) inc += y;
        }
        wcnt[b0 + lane] = carry + inc - v;
        carry += __shfl_sync(0xffffffffu, inc, 31);
      }
      if (lane == 0) wcnt[kBtEmitTiles * kW] = carry;
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < kBtEmitTiles; ++u) {
      const bool f = (flags >> u) & 1u;
      const unsigned bal = __ballot_sync(0xffffffffu, f);
      if (f) {
        const int i = r0 + u * kBtScanT + threadIdx.x;
        out[o_base + wcnt[u * kW + warp] + __popc(bal & ((1u << lane) - 1u))] = src.pos(i);
      }
    }
    o_base += wcnt[kBtEmitTiles * kW];
    __syncthreads();
  }
  if (seg == 0 && threadIdx.x == 0) p.n_sel[row] = K;
}

cudaError_t launch_bt_topk(const SelParams& p, const BtBuf& bt, int rows, cudaStream_t st) {
  cudaError_t e = launch_k(sel_bt_thresh_kernel, dim3(kBtThCS, rows), dim3(kBtThT), 0, st, p, bt);
  if (e == cudaSuccess) e = launch_k(sel_bt_scan_kernel, dim3(bt.P, rows), dim3(kBtScanT), 0, st, p, bt);
  if (e == cudaSuccess) e = launch_k(sel_bt_emit_kernel, dim3(bt.P, rows), dim3(kBtScanT), 0, st, p, bt);
  return e;
}

// ---------------------------------------------------------------------------
// Sequence sharding (C4): candidates of the local top-k, then the global pick.

// (z_adj score, global position) of this shard's local top-k; -inf / 0 pads
__global__ void sel_seq_cand_kernel(const SelParams p, int pos_base, double* cand_score, int32_t* cand_pos) {
  griddep_wait();
  griddep_launch();
  const int row = blockIdx.x;
  const Src<false> src(p, row / p.H);
  const int cnt = p.n_sel[row];
  for (int i = threadIdx.x; i < p.K; i += blockDim.x) {
    double sc = -INFINITY;
    int32_t pos = 0;
    if (i < cnt) {
      const int pl = p.sel[(size_t)row * p.K + i];
      sc = p.sb[(size_t)row * p.ld + (pl - src.j_min)];
      pos = pl + pos_base;
    }
    cand_score[(size_t)row * p.K + i] = sc;
    cand_pos[(size_t)row * p.K + i] = pos;
  }
}

// all-gathered [P][rows][K] scores -> [rows][P*K] (shard order = position order),
// plus the index list 0..P*K-1 the explicit top-k ranks them by
__global__ void sel_seq_gather_kernel(int P, int rows, int K, const double* cand_all, double* scores_t,
                                      int32_t* iota) {
  griddep_wait();
  griddep_launch();
  const int row = blockIdx.y;
  const int n = P * K;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int sh = i / K, k = i % K;
    scores_t[(size_t)row * n + i] = cand_all[((size_t)sh * rows + row) * K + k];
    if (row == 0) iota[i] = i;
  }
}

// global top-k indices (ascending = position order) -> this shard's positions,
// local, ascending, into sel / n_sel; pads (position 0) dropped
constexpr int kPickT = 256;
__global__ void __launch_bounds__(kPickT) sel_seq_pick_kernel(int P, int rows, int K, const int32_t* idx_sel,
                                                               const int32_t* idx_n, const int32_t* cand_pos_all,
                                                               int pos_base, int pos_end, int32_t* sel,
                                                               int32_t* n_sel) {
  griddep_wait();
  griddep_launch();
  __shared__ int wsum[kPickT / 32];
  const int row = blockIdx.x;
  const int cnt = idx_n[row];
  const int per = (K + kPickT - 1) / kPickT;
  const int i0 = threadIdx.x * per;
  int keep = 0;
  for (int i = i0; i < min(cnt, i0 + per); ++i) {
    const int id = idx_sel[(size_t)row * K + i];
    const int pos = cand_pos_all[((size_t)(id / K) * rows + row) * K + (id % K)];
    keep += (pos > pos_base && pos <= pos_end) ? 1 : 0;
  }
  // block exclusive scan of keep
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int x = keep;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wsum[warp] = x;
  __syncthreads();
  int base = 0, total = 0;
  for (int w = 0; w < kPickT / 32; ++w) {
    if (w < warp) base += wsum[w];
    total += wsum[w];
  }
  int o = base + x - keep;
  for (int i = i0; i < min(cnt, i0 + per); ++i) {
    const int id = idx_sel[(size_t)row * K + i];
    const int pos = cand_pos_all[((size_t)(id / K) * rows + row) * K + (id % K)];
    if (pos > pos_base && pos <= pos_end) sel[(size_t)row * K + o++] = pos - pos_base;
  }
  if (threadIdx.x == 0) n_sel[row] = total;
}

// phases: 1 = fuse (z_base), 2 = refine + top-k
template <bool kExp>
cudaError_t run3(const SelParams& p, int rows, int n_max, int batches, cudaStream_t st,
                 int* launches, int phases = 3) {
  const dim3 gc(kCS, (unsigned)rows);
  cudaError_t e = cudaSuccess;
  if (phases & 1) {
    if (p.W == 1 && p.alpha == 1.0)
      e = launch_k(sel_fuse_fast_kernel<kExp>, gc, dim3(kT), 0, st, p);
    else if (p.W > 1)
      e = launch_k(sel_fuse_kernel<kExp, kMaxW>, gc, dim3(kT), 0, st, p);
    else
      e = launch_k(sel_fuse_kernel<kExp, 1>, gc, dim3(kT), 0, st, p);
    if (launches) *launches += 1;
  }
  if (e != cudaSuccess || !(phases & 2)) return e;
  const dim3 gr((n_max + kRefineT - 1) / kRefineT, batches);
  const dim3 br(kRefineT);
  switch (p.z_all ? p.H_all : p.H) {
    case 1: e = launch_k(sel_refine_kernel<kExp, 1>, gr, br, 0, st, p); break;
    case 2: e = launch_k(sel_refine_kernel<kExp, 2>, gr, br, 0, st, p); break;
    case 4: e = launch_k(sel_refine_kernel<kExp, 4>, gr, br, 0, st, p); break;
    case 8: e = launch_k(sel_refine_kernel<kExp, 8>, gr, br, 0, st, p); break;
    default: e = launch_k(sel_refine_kernel<kExp, 16>, gr, br, 0, st, p); break;
  }
  if (e != cudaSuccess) return e;
  e = launch_topk<kExp>(p, rows, n_max, st);
  if (launches) *launches += 2;
  return e;
}

}  // namespace

cudaError_t launch_selector(const sfi_shape& s, const sfi_cache& c, int layer, const float* logits,
                            const sfi_selector_params& prm, const SelectorScratch& scr,
                            cudaStream_t st, int* launches, int phases, const double* z_all,
                            int n_shards, int shard, int W) {
  SelParams p{};
  p.z_all = z_all;
  p.H_all = z_all ? n_shards * s.n_kv_heads : s.n_kv_heads;
  p.h_off = z_all ? shard * s.n_kv_heads : 0;
  if (p.H_all > 16) return cudaErrorInvalidValue;
  const size_t slices = (size_t)s.batch * s.n_kv_heads;
  p.logits32 = logits;
  p.norms_c = c.key_norms + (size_t)layer * slices * s.max_positions;
  p.prefix_len = c.prefix_len;
  p.n_sink_b = c.n_sink_b;
  p.recent_len = c.recent_len;
  p.W = 1;
  p.ld = s.max_positions;
  p.sa = scr.a;
  p.sb = scr.b;
  p.sel = c.sel + (size_t)layer * slices * s.k_budget;
  p.n_sel = c.n_sel + (size_t)layer * slices;
  p.err = c.error_flags;
  p.B = s.batch;
  p.H = s.n_kv_heads;
  p.Lmax = s.max_positions;
  p.K = s.k_budget;
  fill_cfg(p, prm);
  if (s.n_kv_heads > 16) return cudaErrorInvalidValue;
  static const bool legacy = [] {
    const char* e = std::getenv("SFI_SELECTOR_3K");
    return e && e[0] == '1';
  }();
  p.W = W;
  if (phases == 3 && !z_all && W == 1 && p.alpha == 1.0 && p.nms_radius <= kMaxNmsR && !legacy && scr.c) {
    // decode Selector: P/W + chunk statistics, fused z / soft-NMS / cross-head, top-k
    const int ldc = n_chunks(s.max_positions);
    const dim3 gz((s.max_positions + kRefineT - 1) / kRefineT, s.batch);
    const dim3 ba(kPwT), bz(kRefineT);
    double* P = scr.a;
    double* Wt = scr.c;
    double* stt = scr.stats;
    double* cf = scr.stats + slices * ldc * 6;  // [rows][ldc + 2] fused coefficients
    cudaError_t e;
    const bool small_pw = (size_t)ldc * s.batch * ((s.n_kv_heads + kPwHeads - 1) / kPwHeads) < 128;
    const bool def_exp = p.gamma == 1.0 && p.p_curve == 2.0 && p.eta == 0.5;
    // long rows: the rows x segments top-k over sel_z's value histogram
    static const bool force_cluster = std::getenv("SFI_TOPK_CLUSTER") != nullptr;
    static const int bt_env = std::getenv("SFI_TOPK_BT") ? std::atoi(std::getenv("SFI_TOPK_BT")) : -1;
    const bool bt_len = bt_env < 0 ? s.max_positions > kTopkCtaMax : bt_env > 0;
    const bool use_bt = scr.bt != nullptr && bt_len && !force_cluster &&
                        p.alpha_soft >= 0.0 && p.alpha_cross >= 0.0;
    BtBuf bt{};
    if (use_bt) {
      uint8_t* w = static_cast<uint8_t*>(scr.bt);
      bt.hist = reinterpret_cast<uint32_t*>(w);
      w += slices * kBtRow * 4;
      bt.cand = reinterpret_cast<int32_t*>(w);
      w += slices * (size_t)s.max_positions * 4;
      bt.meta = reinterpret_cast<int32_t*>(w);
      w += slices * kBtMeta * 4;
      bt.seg = reinterpret_cast<int32_t*>(w);
      bt.P = (int)std::max<size_t>(1, std::min<size_t>(kBtMaxSeg, (296 + slices - 1) / slices));
      p.bt_hist = bt.hist;
      // z_adj in [log(eps) (1 + alpha_soft + alpha_cross), log(1 + eps)] (margins of 1)
      p.bt_zlo = std::log(p.eps) * (1.0 + p.alpha_soft + p.alpha_cross) - 1.0;
      p.bt_scale = (double)(kBtBins - 1) / (std::log1p(p.eps) + 1.0 - p.bt_zlo);
    }
#define SFI_SEL2(KH)                                                                             \
  e = small_pw ? (def_exp ? launch_k(sel_pw_kernel<KH, 1, true>, dim3(ldc, s.batch, KH == 16 ? s.n_kv_heads : KH), \
                                     ba, 0, st, p, P, Wt, stt, ldc)                                  \
                         : launch_k(sel_pw_kernel<KH, 1>, dim3(ldc, s.batch, KH == 16 ? s.n_kv_heads : KH), ba, \
                                    0, st, p, P, Wt, stt, ldc))                                      \
               : (def_exp ? launch_k(sel_pw_kernel<KH, kPwHeads, true>,                              \
                                     dim3(ldc, s.batch, (KH + kPwHeads - 1) / kPwHeads), ba, 0, st, p, P, Wt, stt, ldc) \
                          : launch_k(sel_pw_kernel<KH>, dim3(ldc, s.batch, (KH + kPwHeads - 1) / kPwHeads), ba, 0, \
                                     st, p, P, Wt, stt, ldc));                                       \
  if (e == cudaSuccess)                                                                              \
    e = ldc > 128 ? launch_k(sel_coef_wide_kernel, dim3((unsigned)slices), dim3(256), 0, st, p,        \
                             (const double*)stt, cf, ldc)                                            \
                  : launch_k(sel_coef_kernel, dim3(((unsigned)slices + 7) / 8), dim3(256), 0, st, p,  \
                             (const double*)stt, cf, ldc);                                           \
  if (e == cudaSuccess) e = launch_k(sel_z_kernel<KH>, gz, bz, 0, st, p, (const double*)stt,           \
                                     (const double*)Wt, (const double*)cf, ldc);
    switch (s.n_kv_heads) {
      case 1: SFI_SEL2(1) break;
      case 2: SFI_SEL2(2) break;
      case 4: SFI_SEL2(4) break;
      case 8: SFI_SEL2(8) break;
      default: SFI_SEL2(16) break;
    }
#undef SFI_SEL2
    if (e != cudaSuccess) return e;
    if (launches) *launches += 3;
    if (use_bt) {
      if (launches) *launches += 3;  // 4 kernels instead of one
      return launch_bt_topk(p, bt, (int)slices, st);
    }
    return launch_topk<false>(p, (int)slices, s.max_positions, st);
  }
  return run3<false>(p, (int)slices, s.max_positions, s.batch, st, launches, phases);
}

namespace {
SelParams seq_params(const sfi_shape& s, const sfi_cache& c, int layer, const float* logits,
                     const sfi_selector_params& prm, const SelectorScratch& scr, const int32_t* j_off,
                     const int32_t* n_glob) {
  SelParams p{};
  const size_t slices = (size_t)s.batch * s.n_kv_heads;
  p.logits32 = logits;
  p.norms_c = c.key_norms + (size_t)layer * slices * s.max_positions;
  p.prefix_len = c.prefix_len;
  p.n_sink_b = c.n_sink_b;
  p.recent_len = c.recent_len;
  p.W = 1;
  p.ld = s.max_positions;
  p.sa = scr.a;
  p.sb = scr.b;
  p.sel = c.sel + (size_t)layer * slices * s.k_budget;
  p.n_sel = c.n_sel + (size_t)layer * slices;
  p.err = c.error_flags;
  p.B = s.batch;
  p.H = s.n_kv_heads;
  p.Lmax = s.max_positions;
  p.K = s.k_budget;
  p.j_off = j_off;
  p.n_glob = n_glob;
  fill_cfg(p, prm);
  return p;
}
}  // namespace

cudaError_t launch_seq_selector_stats(const sfi_shape& s, const sfi_cache& c, int layer, const float* logits,
                                      const sfi_selector_params& prm, const SelectorScratch& scr,
                                      const int32_t* j_off, const int32_t* n_glob, int phase, double* row_stats,
                                      const double* stats_all, int n_shards, double* edges, cudaStream_t st) {
  SelParams p = seq_params(s, c, layer, logits, prm, scr, j_off, n_glob);
  p.seq_phase = phase;
  p.row_stats = row_stats;
  p.stats_all = stats_all;
  p.n_shards = n_shards;
  p.edges = edges;
  const dim3 gc(kCS, (unsigned)(s.batch * s.n_kv_heads));
  return launch_k(sel_fuse_fast_kernel<false>, gc, dim3(kT), 0, st, p);
}

cudaError_t launch_seq_selector_finish(const sfi_shape& s, const sfi_cache& c, int layer,
                                       const sfi_selector_params& prm, const SelectorScratch& scr,
                                       const int32_t* j_off, const int32_t* n_glob, const double* edges_all,
                                       int n_shards, int pos_base, double* cand_score, int32_t* cand_pos,
                                       cudaStream_t st, int* launches) {
  SelParams p = seq_params(s, c, layer, nullptr, prm, scr, j_off, n_glob);
  p.edges_all = edges_all;
  p.n_shards = n_shards;
  const int rows = s.batch * s.n_kv_heads;
  cudaError_t e = run3<false>(p, rows, s.max_positions, s.batch, st, launches, 2);
  if (e != cudaSuccess) return e;
  if (launches) *launches += 1;
  return launch_k(sel_seq_cand_kernel, dim3(rows), dim3(256), 0, st, p, pos_base, cand_score, cand_pos);
}

size_t seq_pick_scratch_bytes(const sfi_shape& s, int n_shards) {
  const size_t rows = (size_t)s.batch * s.n_kv_heads, n = (size_t)n_shards * s.k_budget;
  return rows * n * sizeof(double) + ((n * 4 + 255) / 256) * 256 + rows * s.k_budget * 4 + rows * 4 + 1024;
}

cudaError_t launch_seq_selector_pick(const sfi_shape& s, const sfi_cache& c, int layer, int n_shards,
                                     const double* cand_score_all, const int32_t* cand_pos_all, int pos_base,
                                     int pos_end, void* scratch, cudaStream_t st, int* launches) {
  const int rows = s.batch * s.n_kv_heads, K = s.k_budget, n = n_shards * K;
  const size_t slices = (size_t)rows;
  int32_t* sel = c.sel + (size_t)layer * slices * K;
  int32_t* n_sel = c.n_sel + (size_t)layer * slices;
  if (K == 0) return cudaMemsetAsync(n_sel, 0, rows * sizeof(int32_t), st);
  uint8_t* w = static_cast<uint8_t*>(scratch);
  double* scores_t = reinterpret_cast<double*>(w);
  w += (size_t)rows * n * sizeof(double);
  int32_t* iota = reinterpret_cast<int32_t*>(w);
  w += (((size_t)n * 4 + 255) / 256) * 256;
  int32_t* idx_sel = reinterpret_cast<int32_t*>(w);
  w += (size_t)rows * K * 4;
  int32_t* idx_n = reinterpret_cast<int32_t*>(w);
  cudaError_t e = launch_k(sel_seq_gather_kernel, dim3((n + 255) / 256, rows), dim3(256), 0, st, n_shards, rows,
                           K, cand_score_all, scores_t, iota);
  if (e != cudaSuccess) return e;
  SelParams p{};
  p.allowed = iota;
  p.n_fixed = n;
  p.W = 1;
  p.ld = n;
  p.sb = scores_t;
  p.sel = idx_sel;
  p.n_sel = idx_n;
  p.B = rows;
  p.H = 1;
  p.Lmax = n;
  p.K = K;
  if ((e = launch_topk<true>(p, rows, n, st)) != cudaSuccess) return e;
  if (launches) *launches += 3;
  return launch_k(sel_seq_pick_kernel, dim3(rows), dim3(kPickT), 0, st, n_shards, rows, K,
                  (const int32_t*)idx_sel, (const int32_t*)idx_n, cand_pos_all, pos_base, pos_end, sel, n_sel);
}

cudaError_t launch_selector_explicit(int H, int W, int n, int K, const double* logits, const double* norms,
                                     const int32_t* allowed, const sfi_selector_params& prm, double* sa,
                                     double* sb, int32_t* sel, int32_t* n_sel, uint32_t* err,
                                     cudaStream_t st, int* launches) {
  SelParams p{};
  p.logits64 = logits;
  p.norms_e = norms;
  p.allowed = allowed;
  p.n_fixed = n;
  p.W = W;
  p.ld = n;
  p.sa = sa;
  p.sb = sb;
  p.sel = sel;
  p.n_sel = n_sel;
  p.err = err;
  p.B = 1;
  p.H = H;
  p.Lmax = n;
  p.K = K;
  fill_cfg(p, prm);
  if (H > 16 || W > kMaxW || W < 1) return cudaErrorInvalidValue;
  return run3<true>(p, H, n, 1, st, launches);
}

cudaError_t launch_topk_explicit(int rows, int n, int K, const double* scores, const int32_t* allowed,
                                 int32_t* sel, int32_t* n_sel, cudaStream_t st, int* launches) {
  SelParams p{};
  p.allowed = allowed;
  p.n_fixed = n;
  p.W = 1;
  p.ld = n;
  p.sb = const_cast<double*>(scores);
  p.sel = sel;
  p.n_sel = n_sel;
  p.B = rows;
  p.H = 1;
  p.Lmax = n;
  p.K = K;
  if (launches) *launches += 1;
  return launch_topk<true>(p, rows, n, st);
}

}  // namespace sfi_impl

// ---------------------------------------------------------------------------
// Reference-facing Selector stages (selector.hpp:84-122, distribution.cpp:
// 41-60): one CTA per head row, deterministic block reductions, the
// reference's formulas in its operation order (the stage API is the
// reference's debugging / composition surface; the decode hot path uses the
// fused kernels above). Per-head errors land in head_err[h] (0 = ok, else the
// sfi_status code of the FIRST failure in the reference's check order).
namespace sfi_impl {
namespace {

constexpr int kStageT = 256;

template <typename Op>
__device__ __forceinline__ double stage_reduce(double v, double* red, Op op) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = op(v, __shfl_xor_sync(0xffffffffu, v, o));
  __syncthreads();  // red may still be read by the previous call
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double acc = red[0];
  for (int w = 1; w < kStageT / 32; ++w) acc = op(acc, red[w]);
  return acc;
}

struct StageArgs {
  int H, W, n;
  const double* a;
  const double* b;
  double* out;
  double* out2;
  int32_t* head_err;
  double alpha, gamma, beta, p_curve, eta, lambda_clip, alpha_soft, alpha_cross, temperature, eps;
  int nms_radius;
};

// normalize(weights) of one row in place (distribution.cpp:41-60); false on error
__device__ bool stage_normalize_row(const double* w, double* out, int n, double* red, int32_t* err) {
  bool bad = false;
  double s = 0.0;
  for (int j = threadIdx.x; j < n; j += kStageT) {
    const double x = w[j];
    if (!isfinite(x) || x < 0.0) bad = true;
    s += x;
  }
  const double anybad = stage_reduce(bad ? 1.0 : 0.0, red, OpMax{});
  if (anybad > 0.0) {
    if (threadIdx.x == 0) *err = SFI_ERR_NON_FINITE_INPUT;
    return false;
  }
  const double sum = stage_reduce(s, red, OpSum{});
  if (sum <= 0.0) {
    if (threadIdx.x == 0) *err = SFI_ERR_EMPTY_SUPPORT;
    return false;
  }
  for (int j = threadIdx.x; j < n; j += kStageT) out[j] = w[j] / sum;
  return true;
}

// evidence_from_window (selector.cpp:54-74, 96-127): per window row softmax
// (finite check, max from kMaskedLogit, masked -> 0, sum, divide), power mean
// over the rows, inverse power map, normalize.
__global__ void __launch_bounds__(kStageT) stage_evidence_kernel(const StageArgs p) {
  __shared__ double red[kStageT / 32];
  const int h = blockIdx.x, n = p.n;
  double* mu = p.out + (size_t)h * n;
  for (int row = 0; row < p.W; ++row) {
    const double* v = p.a + ((size_t)h * p.W + row) * n;
    bool bad = false;
    double m = kMaskedLogit;
    for (int j = threadIdx.x; j < n; j += kStageT) {
      const double x = v[j];
      if (!isfinite(x)) bad = true;
      else m = smax(m, x);
    }
    if (stage_reduce(bad ? 1.0 : 0.0, red, OpMax{}) > 0.0) {
      if (threadIdx.x == 0) p.head_err[h] = SFI_ERR_NON_FINITE_INPUT;
      return;
    }
    const double M = stage_reduce(m, red, OpMax{});
    double s = 0.0;
    for (int j = threadIdx.x; j < n; j += kStageT) s += (v[j] <= kMaskedLogit) ? 0.0 : exp(v[j] - M);
    const double sum = stage_reduce(s, red, OpSum{});
    if (sum <= 0.0) {
      if (threadIdx.x == 0) p.head_err[h] = SFI_ERR_EMPTY_SUPPORT;
      return;
    }
    for (int j = threadIdx.x; j < n; j += kStageT) {
      const double pj = ((v[j] <= kMaskedLogit) ? 0.0 : exp(v[j] - M)) / sum;
      mu[j] = (row == 0 ? 0.0 : mu[j]) + pow_ref(pj, p.alpha);
    }
  }
  const double inv_w = 1.0 / (double)p.W;
  const double inv_a = 1.0 / p.alpha;
  for (int j = threadIdx.x; j < n; j += kStageT) mu[j] = pow_ref(mu[j] * inv_w, inv_a);
  __syncthreads();
  stage_normalize_row(mu, mu, n, red, p.head_err + h);
}

// prior_from_stats (selector.cpp:129-160): a = key norms [H][n], b = u(j) [n]
__global__ void __launch_bounds__(kStageT) stage_prior_kernel(const StageArgs p) {
  __shared__ double red[kStageT / 32];
  const int h = blockIdx.x, n = p.n;
  const double* nm = p.a + (size_t)h * n;
  double* w = p.out + (size_t)h * n;
  bool bad = false;
  for (int j = threadIdx.x; j < n; j += kStageT) {
    const double x = nm[j];
    if (!isfinite(x) || x < 0.0) {
      bad = true;
      continue;
    }
    const double u = p.b[j];
    const double pi_kn = pow_ref(x + p.eps, -p.gamma);
    const double pi_pos = exp(-p.beta * pow_ref(u, p.p_curve)) * pow_ref(1.0 - u + p.eps, p.eta);
    w[j] = pi_kn * pi_pos;
  }
  if (stage_reduce(bad ? 1.0 : 0.0, red, OpMax{}) > 0.0) {
    if (threadIdx.x == 0) p.head_err[h] = SFI_ERR_NON_FINITE_INPUT;
    return;
  }
  stage_normalize_row(w, w, n, red, p.head_err + h);
}

__global__ void __launch_bounds__(kStageT) stage_normalize_kernel(const StageArgs p) {
  __shared__ double red[kStageT / 32];
  const int h = blockIdx.x;
  stage_normalize_row(p.a + (size_t)h * p.n, p.out + (size_t)h * p.n, p.n, red, p.head_err + h);
}

// fuse (selector.cpp:162-185): |f|^2, f.r, |r|^2, lambda*, s; out2[h] = lambda*
__global__ void __launch_bounds__(kStageT) stage_fuse_kernel(const StageArgs p) {
  __shared__ double red[kStageT / 32];
  const int h = blockIdx.x, n = p.n;
  const double* f = p.a + (size_t)h * n;
  const double* r = p.b + (size_t)h * n;
  double sff = 0.0, sfr = 0.0, srr = 0.0;
  for (int j = threadIdx.x; j < n; j += kStageT) {
    sff += f[j] * f[j];
    sfr += f[j] * r[j];
    srr += r[j] * r[j];
  }
  const double ff = stage_reduce(sff, red, OpSum{});
  const double fr = stage_reduce(sfr, red, OpSum{});
  const double rr = stage_reduce(srr, red, OpSum{});
  const double denom = ff - 2.0 * fr + rr;
  double lambda = 0.0;
  if (fabs(denom) >= p.eps) {
    lambda = (ff - fr) / denom;
    lambda = (lambda < 0.0) ? 0.0 : (p.lambda_clip < lambda) ? p.lambda_clip : lambda;
  }
  if (threadIdx.x == 0 && p.out2) p.out2[h] = lambda;
  double* s = p.out + (size_t)h * n;
  for (int j = threadIdx.x; j < n; j += kStageT) s[j] = (1.0 - lambda) * f[j] + lambda * r[j];
}

// z = log(s + eps) (selector.cpp:270-276), elementwise over [H][n]
__global__ void stage_zbase_kernel(const StageArgs p) {
  const size_t total = (size_t)p.H * p.n;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x)
    p.out[i] = log(p.a[i] + p.eps);
}

// refine_soft_nms (selector.cpp:187-202) per row, rank-order window
__global__ void stage_soft_nms_kernel(const StageArgs p) {
  const size_t total = (size_t)p.H * p.n;
  const int n = p.n, R = p.nms_radius;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
    const double* z = p.a + (i / n) * n;
    const int j = (int)(i % n);
    const int lo = max(0, j - R), hi = min(n - 1, j + R);
    double m = z[j];
    for (int k = lo; k <= hi; ++k) m = smax(m, z[k]);
    p.out[i] = z[j] - p.alpha_soft * (m - z[j]);
  }
}

// refine_cross_head (selector.cpp:204-230) per position, heads in order
__global__ void stage_cross_head_kernel(const StageArgs p) {
  const int n = p.n, H = p.H;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
    double mx = p.a[j];
    for (int h = 1; h < H; ++h) mx = smax(mx, p.a[(size_t)h * n + j]);
    double sum = 0.0;
    for (int h = 0; h < H; ++h) sum += exp((p.a[(size_t)h * n + j] - mx) / p.temperature);
    for (int h = 0; h < H; ++h) {
      const double z = p.a[(size_t)h * n + j];
      const double r = exp((z - mx) / p.temperature) / sum;
      p.out[(size_t)h * n + j] = z + p.alpha_cross * log(smax(r, p.eps));
    }
  }
}

}  // namespace

cudaError_t launch_selector_stage(int stage, int H, int W, int n, const double* a, const double* b,
                                  const sfi_selector_params& prm, double* out, double* out2, int32_t* head_err,
                                  cudaStream_t st) {
  StageArgs p{};
  p.H = H;
  p.W = W;
  p.n = n;
  p.a = a;
  p.b = b;
  p.out = out;
  p.out2 = out2;
  p.head_err = head_err;
  p.alpha = prm.alpha;
  p.gamma = prm.gamma;
  p.beta = prm.beta;
  p.p_curve = prm.p_curve;
  p.eta = prm.eta;
  p.lambda_clip = prm.lambda_clip;
  p.alpha_soft = prm.alpha_soft;
  p.alpha_cross = prm.alpha_cross;
  p.temperature = prm.temperature;
  p.eps = prm.epsilon;
  p.nms_radius = prm.nms_radius;
  const unsigned elem_blocks = (unsigned)std::min<size_t>(((size_t)H * n + 255) / 256, 4096);
  switch (stage) {
    case SFI_STAGE_EVIDENCE: stage_evidence_kernel<<<H, kStageT, 0, st>>>(p); break;
    case SFI_STAGE_PRIOR: stage_prior_kernel<<<H, kStageT, 0, st>>>(p); break;
    case SFI_STAGE_NORMALIZE: stage_normalize_kernel<<<H, kStageT, 0, st>>>(p); break;
    case SFI_STAGE_FUSE: stage_fuse_kernel<<<H, kStageT, 0, st>>>(p); break;
    case SFI_STAGE_Z_BASE: stage_zbase_kernel<<<std::max(elem_blocks, 1u), 256, 0, st>>>(p); break;
    case SFI_STAGE_SOFT_NMS: stage_soft_nms_kernel<<<std::max(elem_blocks, 1u), 256, 0, st>>>(p); break;
    case SFI_STAGE_CROSS_HEAD:
      stage_cross_head_kernel<<<std::max(std::min((n + 255) / 256, 4096), 1), 256, 0, st>>>(p);
      break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

}  // namespace sfi_impl

// decode.cu — K1 slow-step dense decode (+ pooled-logit emission) and K4
// fast-step sparse decode over the compact cache. One kernel template serves
// both: a (b, kv-head) slice is a list of <= 3 contiguous row segments of a
// bf16 [rows][D] matrix (paged cache for dense; ring + sink/selected rows of
// the compact cache for sparse), cut into 64-row tiles.
//
// Reference semantics (paths relative to /root/reference/proj):
//   attend                attention.cpp:80-113   softmax(q.k / sqrt(d)) v
//   dense_segments        attention.cpp:258-268  positions 1..L (current included)
//   sparse_segments       attention.cpp:270-291  compact + recent rows
//   logit capture / pool  attention.cpp:394-409  mean: sum_g logit_g / G; max
//
// B200 design:
//   * stream-K schedule: the tiles of all slices form one list; CTA c takes
//     the balanced contiguous range [c T / G, (c+1) T / G) (G = 2 CTAs per SM),
//     so every SM streams the same number of bytes whatever the per-slice
//     lengths; a CTA crosses slice boundaries without draining its pipeline
//     and emits at most two partial (m, l, O) results (its first and last
//     slice); slices touched by one CTA are finalised directly, the others by
//     the last-arriving contributor (log-sum-exp merge in CTA order);
//   * a producer warp streams K and V tiles HBM -> smem with TMA
//     (cp.async.bulk.tensor, 128B swizzle, L2 evict-first) through a
//     3-stage mbarrier ring;
//   * 4 consumer warps each own 16 keys of every tile and run QK^T and PV on
//     the tensor cores (mma.sync m16n8k16 bf16 -> fp32). Query rows are the G
//     heads of the GQA group; the hi and lo bf16 halves of q (and of p) fill
//     the otherwise-padded rows 8..15, so fp32 inputs keep ~16 mantissa bits
//     at no extra instruction cost;
//   * online softmax in the log2 domain with quad shuffles; pooled logits are
//     reduced across the group with 3 butterfly shuffles and stored once.
#include <cuda.h>

#include <algorithm>
#include <cmath>
#include <type_traits>

#include "common.cuh"
#include "kernels.h"

namespace sfi_impl {

using namespace sfi_dev;

namespace {

constexpr int kTile = 64;   // keys per pipeline stage
constexpr int kNcw = 4;     // consumer warps (16 keys of each tile each)
constexpr int kThreads = (kNcw + 2) * 32;   // + TMA producer warp + epilogue warp
constexpr int kBarThreads = (kNcw + 1) * 32; // consumers + epilogue on the hand-off barriers
constexpr int kMaxSlices = 4096;

// G = 16 holds 2x the consumer partials: 2 stages keep 2 CTAs per SM
template <int G>
__host__ __device__ constexpr int stages_for() { return G == 16 ? 2 : 3; }

template <int D, int G>
struct Geo {
  static constexpr int kStages = stages_for<G>();
  static constexpr int kBoxes = D / 64;                   // 128-byte TMA boxes per row
  static constexpr int kBoxBytes = kTile * 128;           // 8 KB
  static constexpr int kTileBytes = kBoxes * kBoxBytes;   // one tensor, one tile
  static constexpr int kStageBytes = 2 * kTileBytes;      // K + V
  static constexpr int kRing = kStages * kStageBytes;
};
// rows of one published partial (m, l, O): 8, or 16 for G = 16
template <int G>
__host__ __device__ constexpr int part_rows() { return G > 8 ? 16 : 8; }

// consumer -> epilogue hand-off: per consumer warp G rows of O plus (m, l)
// for 8 rows. The 8-float column chunks of row g are XOR-swizzled by g so the
// float2 stores from the mma layout (8 rows x 4 lanes) are conflict-free
// without padding (padding would cost G = 8 its second CTA per SM).
template <int D, int G>
struct Comb {
  static constexpr int kOFloats = kNcw * G * D;
  static constexpr int kBytes = kOFloats * 4 + kNcw * 2 * G * 4;
  static constexpr int kSmemFixed = Geo<D, G>::kRing + kBytes + 64 /*barriers*/;
};
template <int D>
__device__ __forceinline__ int comb_col(int col, int g) { return col ^ ((g << 3) & (D - 1)); }

struct Slice {
  int off[3];
  int cnt[3];
  int row_base;   // first row of the (layer, b, h) slice in the 2D tensor
  int j_min, j_max;
};

__device__ __forceinline__ int seg_tiles(int c) { return (c + kTile - 1) / kTile; }

// natural-log LSE of a (m, l) pair whose m is in the log2 domain
__device__ __forceinline__ float lse_of(float m, float l) {
  return l > 0.f ? (m + __log2f(l)) * 0.69314718055994531f : -INFINITY;
}

// 128B-swizzled address of 16-byte chunk `chunk` (8 bf16) of tile row `row`.
template <int D>
__device__ __forceinline__ uint32_t swz(uint32_t base, int row, int chunk) {
  return base + (chunk >> 3) * (kTile * 128) + row * 128 + (((chunk & 7) ^ (row & 7)) << 4);
}

// Segments are fixed slots (0: ring part 1, 1: ring wrap, 2: sink+selected)
// with count 0 when absent, so every index below is a compile-time constant.
__device__ __forceinline__ Slice make_slice(const DecodeParams& p, int s, bool flag_errors) {
  Slice sl;
  const int b = s / p.H, h = s % p.H;
  const int L = p.prefix_len[b];
  const int nsb = p.n_sink_b[b];
  const int rl = p.recent_len[b];
  sl.j_min = nsb + 1;
  sl.j_max = L - rl;
  sl.off[0] = sl.off[1] = sl.off[2] = 0;
  sl.cnt[0] = sl.cnt[1] = sl.cnt[2] = 0;
  if (!p.sparse) {
    sl.row_base = ((p.layer * p.B + b) * p.H + h) * p.Lmax;
    sl.cnt[0] = L > 0 ? L : 0;
  } else {
    sl.row_base = ((p.layer * p.B + b) * p.H + h) * p.crows;
    if (rl > 0) {
      const int s0 = (L - rl) % p.R;  // ring slot of recent_start = L - rl + 1
      const int first = min(rl, p.R - s0);
      sl.off[0] = s0;
      sl.cnt[0] = first;
      sl.cnt[1] = rl - first;
    }
    sl.off[2] = p.R;
    sl.cnt[2] = nsb + p.n_sel[(p.layer * p.B + b) * p.H + h];
    if (rl > p.R || sl.cnt[2] > p.crows - p.R) {  // outside the compact layout
      sl.cnt[0] = sl.cnt[1] = sl.cnt[2] = 0;
      if (flag_errors) raise_error(p.err, SFI_ERR_CONFIG);
    }
  }
  return sl;
}

__device__ __forceinline__ int slice_tiles(const Slice& s) {
  return seg_tiles(s.cnt[0]) + seg_tiles(s.cnt[1]) + seg_tiles(s.cnt[2]);
}

// tile index within the slice -> (row offset within slice, valid rows)
__device__ __forceinline__ void tile_at(const Slice& s, int t, int& off, int& nvalid) {
  off = 0;
  nvalid = 0;
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const int nt = seg_tiles(s.cnt[i]);
    if (t >= 0 && t < nt) {
      off = s.off[i] + t * kTile;
      nvalid = min(kTile, s.cnt[i] - t * kTile);
    }
    t -= nt;
  }
}

// first tile of CTA c under the balanced split of T tiles over G CTAs
// (c*T < 2^53 is exact in fp64 and the quotient is either an exact integer
// or >= 1/G away from one, so truncation equals the integer floor.)
__device__ __forceinline__ int cta_start(int c, int T, int G) {
  return (int)(((double)c * (double)T) / (double)G);
}
// the CTA whose range holds tile t (largest c with start(c) <= t)
__device__ __forceinline__ int cta_of(int t, int T, int G) {
  return (int)((((long long)t + 1) * G - 1) / T);
}
// slice holding global tile t: last s with pref[s] <= t
__device__ __forceinline__ int slice_of(const int* pref, int S, int t) {
  int lo = 0, hi = S - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (pref[mid] <= t) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

// Last-arriving contributor of slice s: merge the partials of the non-empty
// CTAs in [c_first, c_last] in CTA order (deterministic) and write the G
// output rows. One pass per chunk of 4 rows: lanes load (m, l) of one
// contributor each (32 at a time, running max with rescaling across batches),
// then every lane streams its D/32 columns of the rows for four contributors
// per iteration so loads stay in flight instead of serialising on L2 latency.
template <int D, int G>
__device__ __noinline__ void merge_slice(const DecodeParams& p, float* outp, float* lse, int P0, int c_first,
                                         int c_last, int T, int Gc, int lane) {
  constexpr int kCols = D / 32;
  constexpr int kGB = G < 4 ? G : 4;
  // contributors per load batch: as many loads in flight as the registers allow
  constexpr int kCB = kGB <= 1 ? 16 : (kGB == 2 ? 8 : 4);
  constexpr int PR = part_rows<G>();
  using Vec = typename std::conditional<kCols == 4, float4, float2>::type;
#pragma unroll
  for (int g0 = 0; g0 < G; g0 += kGB) {
    float acc[kGB][kCols];
    float L[kGB], M[kGB];
#pragma unroll
    for (int gg = 0; gg < kGB; ++gg) {
      L[gg] = 0.f;
      M[gg] = -INFINITY;
#pragma unroll
      for (int k = 0; k < kCols; ++k) acc[gg][k] = 0.f;
    }
    for (int cb = c_first; cb <= c_last; cb += 32) {
      const int c = cb + lane;
      const int c0s = c <= c_last ? cta_start(c, T, Gc) : 0;
      const bool ok = c <= c_last && c0s < cta_start(c + 1, T, Gc);
      const int pc = c * 2 + (c0s >= P0 ? 0 : 1);
      float mi[kGB], li[kGB], sc[kGB];
#pragma unroll
      for (int gg = 0; gg < kGB; ++gg) {
        mi[gg] = ok ? __ldcg(&p.part_ml[((size_t)pc * 2 + 0) * PR + g0 + gg]) : -INFINITY;
        li[gg] = ok ? __ldcg(&p.part_ml[((size_t)pc * 2 + 1) * PR + g0 + gg]) : 0.f;
      }
#pragma unroll
      for (int gg = 0; gg < kGB; ++gg) {
        float mb = mi[gg];
#pragma unroll
        for (int o2 = 16; o2 > 0; o2 >>= 1) mb = fmaxf(mb, __shfl_xor_sync(0xffffffffu, mb, o2));
        const float Mn = fmaxf(M[gg], mb);
        const float Mu = (Mn == -INFINITY) ? 0.f : Mn;
        const float r = fast_exp2(M[gg] - Mu);  // rescale of earlier batches (0 when none)
#pragma unroll
        for (int k = 0; k < kCols; ++k) acc[gg][k] *= r;
        sc[gg] = ok ? fast_exp2(mi[gg] - Mu) : 0.f;
        float lw = li[gg] * sc[gg];
#pragma unroll
        for (int o2 = 16; o2 > 0; o2 >>= 1) lw += __shfl_xor_sync(0xffffffffu, lw, o2);
        L[gg] = L[gg] * r + lw;
        M[gg] = Mn;
      }
      unsigned mask = __ballot_sync(0xffffffffu, ok);
      while (mask) {  // contributors of this batch, kCB at a time, ascending
        int src[kCB];
        bool has[kCB];
#pragma unroll
        for (int j = 0; j < kCB; ++j) {
          has[j] = mask != 0;
          src[j] = has[j] ? __ffs(mask) - 1 : src[0];
          if (has[j]) mask &= mask - 1;
        }
        Vec x[kCB][kGB];
#pragma unroll
        for (int j = 0; j < kCB; ++j) {
          const int pj = __shfl_sync(0xffffffffu, pc, src[j]);
#pragma unroll
          for (int gg = 0; gg < kGB; ++gg)
            x[j][gg] = __ldcg(reinterpret_cast<const Vec*>(p.part_o + ((size_t)pj * PR + g0 + gg) * D) + lane);
        }
#pragma unroll
        for (int j = 0; j < kCB; ++j)
#pragma unroll
          for (int gg = 0; gg < kGB; ++gg) {
            const float sv = __shfl_sync(0xffffffffu, sc[gg], src[j]);
            const float sj = has[j] ? sv : 0.f;
            acc[gg][0] += x[j][gg].x * sj;
            acc[gg][1] += x[j][gg].y * sj;
            if constexpr (kCols == 4) {
              acc[gg][2 % kCols] += x[j][gg].z * sj;
              acc[gg][3 % kCols] += x[j][gg].w * sj;
            }
          }
      }
    }
#pragma unroll
    for (int gg = 0; gg < kGB; ++gg) {
      const float inv = L[gg] > 0.f ? 1.f / L[gg] : 0.f;
      Vec r;
      r.x = acc[gg][0] * inv;
      r.y = acc[gg][1] * inv;
      if constexpr (kCols == 4) {
        r.z = acc[gg][2 % kCols] * inv;
        r.w = acc[gg][3 % kCols] * inv;
      }
      reinterpret_cast<Vec*>(outp + (g0 + gg) * D)[lane] = r;
      if (lse && lane == 0) lse[g0 + gg] = lse_of(M[gg], L[gg]);
    }
  }
}

template <int D, int G>
__global__ void __launch_bounds__(kThreads, 2)
    decode_kernel(const __grid_constant__ CUtensorMap tmk, const __grid_constant__ CUtensorMap tmv,
                  const DecodeParams p) {
  static_assert(G == 1 || G == 2 || G == 4 || G == 8 || G == 16, "GQA group 1..16");
  static_assert(D == 64 || D == 128, "head_dim 64 or 128");
  constexpr int NH = (G == 16) ? 2 : 1;   // query heads per mma row-thread
  constexpr int NQ = (G == 16) ? 2 : 1;   // A-operand blocks (hi / lo) per k-step
  constexpr int PR = part_rows<G>();
  constexpr int kStages = Geo<D, G>::kStages;
  // 1024-byte alignment (128B-swizzled TMA boxes) without padding slack: the
  // kernel has no static shared memory, so the dynamic window starts at 0
  extern __shared__ __align__(1024) uint8_t smem[];
  float* comb_o = reinterpret_cast<float*>(smem + Geo<D, G>::kRing);        // [kNcw][G][kRow]
  float* comb_ml = comb_o + Comb<D, G>::kOFloats;                           // [kNcw][2][G]
  uint64_t* full = reinterpret_cast<uint64_t*>(comb_ml + kNcw * 2 * G);
  uint64_t* empty = full + kStages;
  int* pref = reinterpret_cast<int*>(empty + kStages + 2);                  // [S + 1]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int S = p.B * p.H;
  long long* trace = p.trace ? p.trace + (size_t)blockIdx.x * 16 : nullptr;
  if (trace && threadIdx.x == 0) {
    trace[0] = (long long)globaltimer();
    trace[6] = smid();
  }

  if (threadIdx.x == kNcw * 32) {  // descriptors are launch constants: fetch before the wait
    tma_prefetch_desc(&tmk);
    tma_prefetch_desc(&tmv);
  }
  // PDL: lengths, selections and the freshly appended ring row are all
  // produced upstream in the same stream
  griddep_wait();
  griddep_launch();

  // ---- per-slice tile counts -> exclusive prefix (every CTA, S <= kMaxSlices) ----
  for (int s = threadIdx.x; s < S; s += kThreads) {
    const Slice sl = make_slice(p, s, blockIdx.x == 0);
    const int n = slice_tiles(sl);
    pref[s + 1] = n;
    if (n == 0 && blockIdx.x == 0) {
      if (p.lse) {  // partial mode (sequence shard without rows): O = 0, lse = -inf
        const int b = s / p.H, h = s % p.H;
        for (int i = 0; i < G * D; ++i) p.out[((size_t)b * p.Hq + (size_t)h * G) * D + i] = 0.f;
        for (int gg = 0; gg < G; ++gg) p.lse[(size_t)b * p.Hq + (size_t)h * G + gg] = -INFINITY;
      } else {
        raise_error(p.err, SFI_ERR_EMPTY_SUPPORT);
      }
    }
  }
  if (threadIdx.x == 0) {
    pref[0] = 0;
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kNcw);
    }
    fence_barrier_init();
  }
  __syncthreads();
  if (warp == 0) {  // inclusive scan of pref[1..S] in chunks of 32
    int carry = 0;
    for (int base = 1; base <= S; base += 32) {
      const int i = base + lane;
      int v = (i <= S) ? pref[i] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += y;
      }
      if (i <= S) pref[i] = v + carry;
      carry += __shfl_sync(0xffffffffu, v, 31);
    }
  }
  __syncthreads();
  const int T = pref[S];
  const int Gc = gridDim.x;
  const int tb = cta_start(blockIdx.x, T, Gc);
  const int te = cta_start(blockIdx.x + 1, T, Gc);
  if (tb >= te) return;  // no tiles for this CTA
  const int s_first = slice_of(pref, S, tb);
  if (trace && threadIdx.x == 0) {
    trace[1] = (long long)globaltimer();
    trace[5] = te - tb;
  }

  if (warp == kNcw) {
    // ---------------- producer: TMA K/V tiles into the stage ring ----------------
    if (lane == 0) {
      const uint64_t pol = l2_policy_evict_first();
      int s = s_first;
      Slice sl = make_slice(p, s, false);
      for (int t = tb, i = 0; t < te; ++t, ++i) {
        while (pref[s + 1] <= t) sl = make_slice(p, ++s, false);
        const int st = i % kStages;
        const uint32_t ph = (i / kStages) & 1;
        mbar_wait(&empty[st], ph ^ 1);
        int off, nv;
        tile_at(sl, t - pref[s], off, nv);
        const int row = sl.row_base + off;
        uint8_t* kdst = smem + st * Geo<D, G>::kStageBytes;
        uint8_t* vdst = kdst + Geo<D, G>::kTileBytes;
        mbar_arrive_expect_tx(&full[st], Geo<D, G>::kStageBytes);
#pragma unroll
        for (int bx = 0; bx < Geo<D, G>::kBoxes; ++bx) {
          tma_load_2d(kdst + bx * Geo<D, G>::kBoxBytes, &tmk, bx * 64, row, &full[st], pol);
          tma_load_2d(vdst + bx * Geo<D, G>::kBoxBytes, &tmv, bx * 64, row, &full[st], pol);
        }
      }
    }
    return;
  }

  if (warp == kNcw + 1) {
    // ---------------- epilogue: combine the 4 consumer partials, emit ----------------
    // Lane l owns columns [l * D/32, (l + 1) * D/32) of every query row. The
    // emission sequence is the CTA's non-empty slices in order, the same
    // sequence the consumers walk.
    constexpr int kCols = D / 32;
    using Vec = typename std::conditional<kCols == 4, float4, float2>::type;
    named_bar_arrive<2, kBarThreads>();  // slots start free
    int pend[2], n_pend = 0;  // partial slices awaiting publication
    for (int s = s_first; s < S && pref[s] < te; ++s) {
      const int P0 = pref[s], P1 = pref[s + 1];
      if (P1 == P0) continue;
      named_bar_sync<1, kBarThreads>();
      const long long e0 = trace ? (long long)globaltimer() : 0;
      if (trace && lane == 0) {
        if (trace[13] == 0) trace[13] = e0;
        trace[14] = e0;
      }
      Vec acc[G];
      float mr[G], lr[G];
#pragma unroll
      for (int gg = 0; gg < G; ++gg) {
        float mw[kNcw], M = -INFINITY;
#pragma unroll
        for (int w = 0; w < kNcw; ++w) {
          mw[w] = comb_ml[(w * 2 + 0) * G + gg];
          M = fmaxf(M, mw[w]);
        }
        const float Mu = (M == -INFINITY) ? 0.f : M;
        float L = 0.f;
        Vec a;
        a.x = a.y = 0.f;
        if constexpr (kCols == 4) a.z = a.w = 0.f;
#pragma unroll
        for (int w = 0; w < kNcw; ++w) {
          const float sc = fast_exp2(mw[w] - Mu);
          L += comb_ml[(w * 2 + 1) * G + gg] * sc;
          const Vec x = *reinterpret_cast<const Vec*>(comb_o + (w * G + gg) * D +
                                                      comb_col<D>(lane * kCols, gg));
          a.x += x.x * sc;
          a.y += x.y * sc;
          if constexpr (kCols == 4) {
            a.z += x.z * sc;
            a.w += x.w * sc;
          }
        }
        acc[gg] = a;
        mr[gg] = M;
        lr[gg] = L;
      }
      __syncwarp();
      named_bar_arrive<2, kBarThreads>();  // slots free again
      const int c_first = cta_of(P0, T, Gc), c_last = cta_of(P1 - 1, T, Gc);
      const int b = s / p.H, h = s % p.H;
      float* outp = p.out + ((size_t)b * p.Hq + (size_t)h * G) * D;
      if (c_first == c_last) {
#pragma unroll
        for (int gg = 0; gg < G; ++gg) {
          const float inv = lr[gg] > 0.f ? 1.f / lr[gg] : 0.f;
          Vec r = acc[gg];
          r.x *= inv;
          r.y *= inv;
          if constexpr (kCols == 4) {
            r.z *= inv;
            r.w *= inv;
          }
          reinterpret_cast<Vec*>(outp + gg * D)[lane] = r;
          if (p.lse && lane == gg) p.lse[(size_t)b * p.Hq + (size_t)h * G + gg] = lse_of(mr[gg], lr[gg]);
        }
      } else {
        // partial: written now, published (fence + counter) once this CTA's
        // stream has ended — a fence issued while the producer's TMA loads are
        // in flight stalls until they drain
        const int slot = (s == s_first) ? 0 : 1;
        const size_t part = (size_t)blockIdx.x * 2 + slot;
#pragma unroll
        for (int gg = 0; gg < G; ++gg) {
          reinterpret_cast<Vec*>(p.part_o + (part * PR + gg) * D)[lane] = acc[gg];
          if (lane == gg) {
            p.part_ml[(part * 2 + 0) * PR + gg] = mr[gg];
            p.part_ml[(part * 2 + 1) * PR + gg] = lr[gg];
          }
        }
        pend[n_pend++] = s;
      }
      if (trace && lane == 0) {
        trace[4] += 1;  // emissions
        trace[7] += (long long)globaltimer() - e0;
      }
    }
    if (n_pend > 0) {
      const long long e1 = trace ? (long long)globaltimer() : 0;
      __threadfence();  // release this CTA's partials
      __syncwarp();
      if (trace && lane == 0) trace[9] = (long long)globaltimer() - e1;
      for (int k = 0; k < n_pend; ++k) {
        const int sp = pend[k];
        const int P0 = pref[sp], P1 = pref[sp + 1];
        const int c_first = cta_of(P0, T, Gc), c_last = cta_of(P1 - 1, T, Gc);
        // contributors = CTAs in [c_first, c_last] with a non-empty range
        int n_contrib = 0;
        for (int cb = c_first; cb <= c_last; cb += 32) {
          const int c = cb + lane;
          const bool ok = c <= c_last && cta_start(c, T, Gc) < cta_start(c + 1, T, Gc);
          n_contrib += __popc(__ballot_sync(0xffffffffu, ok));
        }
        int last = 0;
        if (lane == 0) last = (atomicAdd(&p.counters[sp], 1) == n_contrib - 1);
        last = __shfl_sync(0xffffffffu, last, 0);
        if (last) {
          __threadfence();  // acquire the other contributors' partials
          const int b = sp / p.H, h = sp % p.H;
          merge_slice<D, G>(p, p.out + ((size_t)b * p.Hq + (size_t)h * G) * D,
                            p.lse ? p.lse + (size_t)b * p.Hq + (size_t)h * G : nullptr, P0, c_first, c_last,
                            T, Gc, lane);
          if (lane == 0) p.counters[sp] = 0;
        }
      }
      if (trace && lane == 0) trace[10] += (long long)globaltimer() - e1;
    }
    if (trace && lane == 0) trace[3] = (long long)globaltimer();
    return;
  }

  // ---------------- consumers ----------------
  const int g = lane >> 2, t4 = lane & 3;
  const float sl2 = p.scale_log2;
  uint32_t qa[NQ][D / 16][4];
  float o[D / 8][4];
  float m_run[NH], l_run[NH];
  int s = s_first;
  Slice sl = make_slice(p, s, false);
  bool fresh = true;

  for (int t = tb, i = 0; t < te; ++t, ++i) {
    while (pref[s + 1] <= t) sl = make_slice(p, ++s, false);
    if (fresh) {
      // Q fragments. G <= 8: rows 0..7 = bf16 hi of head g (< G), rows 8..15 = lo.
      // G == 16: block 0 = hi of heads 0..15, block 1 = lo.
      const int b = s / p.H, h = s % p.H;
      const float* qb = p.q + ((size_t)b * p.Hq + (size_t)h * G) * D;
#pragma unroll
      for (int ks = 0; ks < D / 16; ++ks) {
#pragma unroll
        for (int half = 0; half < 2; ++half) {
          const int c = ks * 16 + half * 8 + 2 * t4;
          if constexpr (G == 16) {
#pragma unroll
            for (int r = 0; r < 2; ++r) {
              const float2 v = *reinterpret_cast<const float2*>(qb + (g + 8 * r) * D + c);
              float h0, l0, h1, l1;
              split_bf16(v.x, h0, l0);
              split_bf16(v.y, h1, l1);
              qa[0][ks][half * 2 + r] = pack_bf16(h0, h1);
              qa[NQ - 1][ks][half * 2 + r] = pack_bf16(l0, l1);
            }
          } else {
            float x0 = 0.f, x1 = 0.f;
            if (g < G) {
              const float2 v = *reinterpret_cast<const float2*>(qb + g * D + c);
              x0 = v.x;
              x1 = v.y;
            }
            float h0, l0, h1, l1;
            split_bf16(x0, h0, l0);
            split_bf16(x1, h1, l1);
            qa[0][ks][half * 2 + 0] = pack_bf16(h0, h1);
            qa[0][ks][half * 2 + 1] = pack_bf16(l0, l1);
          }
        }
      }
#pragma unroll
      for (int n = 0; n < D / 8; ++n) o[n][0] = o[n][1] = o[n][2] = o[n][3] = 0.f;
#pragma unroll
      for (int hh = 0; hh < NH; ++hh) {
        m_run[hh] = -INFINITY;
        l_run[hh] = 0.f;
      }
      fresh = false;
    }
    const int st = i % kStages;
    const uint32_t ph = (i / kStages) & 1;
    int off, nv;
    tile_at(sl, t - pref[s], off, nv);
    mbar_wait(&full[st], ph);
    if (trace && i == 0 && threadIdx.x == 0) trace[2] = (long long)globaltimer();
    const int kw = warp * 16;  // this warp's first key in the tile
    if (kw < nv) {
      const uint32_t kbase = smem_u32(smem + st * Geo<D, G>::kStageBytes);
      const uint32_t vbase = kbase + Geo<D, G>::kTileBytes;
      // ---- S = Q K^T for 16 keys ----
      // G = 16: the hi and lo query blocks accumulate in separate chains (2x the
      // independent HMMA chains), summed once
      float acc[2][4], acc_lo[2][4];
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.f;
        acc_lo[j][0] = acc_lo[j][1] = acc_lo[j][2] = acc_lo[j][3] = 0.f;
      }
#pragma unroll
      for (int kc = 0; kc < D / 16; kc += 2) {
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          uint32_t b0, b1, b2, b3;
          ldsm_x4(swz<D>(kbase, kw + j * 8 + (lane & 7), kc * 2 + (lane >> 3)), b0, b1, b2, b3);
          mma_bf16(acc[j], qa[0][kc], b0, b1);
          mma_bf16(acc[j], qa[0][kc + 1], b2, b3);
          if constexpr (NQ == 2) {
            mma_bf16(acc_lo[j], qa[NQ - 1][kc], b0, b1);
            mma_bf16(acc_lo[j], qa[NQ - 1][kc + 1], b2, b3);
          }
        }
      }
      if constexpr (NQ == 2) {
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
          for (int e = 0; e < 4; ++e) acc[j][e] += acc_lo[j][e];
      }
      float sc[NH][2][2];
      bool valid[2][2];
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          if constexpr (NH == 2) {
            sc[0][j][e] = acc[j][e];
            sc[NH - 1][j][e] = acc[j][e + 2];
          } else {
            sc[0][j][e] = acc[j][e] + acc[j][e + 2];
          }
          valid[j][e] = (kw + j * 8 + 2 * t4 + e) < nv;
        }
      // ---- pooled logits over J (dense slow step) ----
      if (p.logits != nullptr) {
        const int pos0 = off + kw + 1;  // dense row r holds position r + 1
        if (pos0 + 15 >= sl.j_min && pos0 <= sl.j_max) {
#pragma unroll
          for (int j = 0; j < 2; ++j)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              float v;
              if (p.pool == SFI_POOL_MAX) {
                v = (NH == 2 || g < G) ? sc[0][j][e] * p.inv_sqrt_d : -INFINITY;
                if constexpr (NH == 2) v = fmaxf(v, sc[NH - 1][j][e] * p.inv_sqrt_d);
                v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, 4));
                v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, 8));
                v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, 16));
              } else {
                v = sc[0][j][e] * p.inv_sqrt_d;
                if constexpr (NH == 2) v += sc[NH - 1][j][e] * p.inv_sqrt_d;
                v += __shfl_xor_sync(0xffffffffu, v, 4);
                v += __shfl_xor_sync(0xffffffffu, v, 8);
                v += __shfl_xor_sync(0xffffffffu, v, 16);
                v *= (1.0f / G);
              }
              const int pos = pos0 + j * 8 + 2 * t4 + e;
              if (g == 0 && valid[j][e] && pos >= sl.j_min && pos <= sl.j_max)
                p.logits[(size_t)s * p.Lmax + (pos - sl.j_min)] = v;
            }
        }
      }
      // ---- online softmax (log2 domain) ----
      float pr[NH][2][2], alpha[NH];
      bool any_grow = false;
#pragma unroll
      for (int hh = 0; hh < NH; ++hh) {
        float mx = -INFINITY;
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            sc[hh][j][e] = valid[j][e] ? sc[hh][j][e] * sl2 : -INFINITY;
            mx = fmaxf(mx, sc[hh][j][e]);
          }
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
        // lazy rescaling: the reference max moves only when the tile's max
        // exceeds it by more than 2^8 (p <= 256 otherwise; (m, l, O) stay a
        // consistent triple), so O is rarely rescaled
        const bool grow = mx > m_run[hh] + kLazyMax;
        const float m_new = grow ? mx : m_run[hh];
        const float m_use = (m_new == -INFINITY) ? 0.f : m_new;
        alpha[hh] = grow ? fast_exp2(m_run[hh] - m_use) : 1.f;
        any_grow |= grow;
        float psum = 0.f;
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            pr[hh][j][e] = fast_exp2(sc[hh][j][e] - m_use);
            psum += pr[hh][j][e];
          }
        l_run[hh] = l_run[hh] * alpha[hh] + psum;
        m_run[hh] = m_new;
      }
      if (__any_sync(0xffffffffu, any_grow)) {
#pragma unroll
        for (int n = 0; n < D / 8; ++n) {
          o[n][0] *= alpha[0];
          o[n][1] *= alpha[0];
          o[n][2] *= alpha[NH - 1];
          o[n][3] *= alpha[NH - 1];
        }
      }
      // ---- P as the A operand (rows as the Q fragments) ----
      uint32_t pa[NQ][4];
      {
        float hi[NH][2][2], lo[NH][2][2];
#pragma unroll
        for (int hh = 0; hh < NH; ++hh)
#pragma unroll
          for (int j = 0; j < 2; ++j)
#pragma unroll
            for (int e = 0; e < 2; ++e) split_bf16(pr[hh][j][e], hi[hh][j][e], lo[hh][j][e]);
        if constexpr (NH == 2) {
          pa[0][0] = pack_bf16(hi[0][0][0], hi[0][0][1]);
          pa[0][1] = pack_bf16(hi[1][0][0], hi[1][0][1]);
          pa[0][2] = pack_bf16(hi[0][1][0], hi[0][1][1]);
          pa[0][3] = pack_bf16(hi[1][1][0], hi[1][1][1]);
          pa[NQ - 1][0] = pack_bf16(lo[0][0][0], lo[0][0][1]);
          pa[NQ - 1][1] = pack_bf16(lo[1][0][0], lo[1][0][1]);
          pa[NQ - 1][2] = pack_bf16(lo[0][1][0], lo[0][1][1]);
          pa[NQ - 1][3] = pack_bf16(lo[1][1][0], lo[1][1][1]);
        } else {
          pa[0][0] = pack_bf16(hi[0][0][0], hi[0][0][1]);
          pa[0][1] = pack_bf16(lo[0][0][0], lo[0][0][1]);
          pa[0][2] = pack_bf16(hi[0][1][0], hi[0][1][1]);
          pa[0][3] = pack_bf16(lo[0][1][0], lo[0][1][1]);
        }
      }
      // ---- O += P V ----
#pragma unroll
      for (int nd = 0; nd < D / 8; nd += 2) {
        const int mi = lane >> 3;
        uint32_t v0, v1, v2, v3;
        ldsm_x4_t(swz<D>(vbase, kw + (mi & 1) * 8 + (lane & 7), nd + (mi >> 1)), v0, v1, v2, v3);
#pragma unroll
        for (int qb = 0; qb < NQ; ++qb) {
          mma_bf16(o[nd], pa[qb], v0, v1);
          mma_bf16(o[nd + 1], pa[qb], v2, v3);
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);

    // ---- end of this CTA's part of slice s: hand the warp partial to the
    // epilogue warp and keep consuming: EMPTY (barrier 2) -> slot -> FULL (barrier 1)
    if (t + 1 == pref[s + 1] || t + 1 == te) {
      float lr[NH];
#pragma unroll
      for (int hh = 0; hh < NH; ++hh) {
        lr[hh] = l_run[hh];
        lr[hh] += __shfl_xor_sync(0xffffffffu, lr[hh], 1);
        lr[hh] += __shfl_xor_sync(0xffffffffu, lr[hh], 2);
      }
      const long long tw0 = trace ? (long long)globaltimer() : 0;
      named_bar_sync<2, kBarThreads>();
      if (trace && threadIdx.x == 0) trace[8] += (long long)globaltimer() - tw0;
      if constexpr (NH == 2) {
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          const int row = g + 8 * hh;
          float* dst = comb_o + (warp * G + row) * D;
#pragma unroll
          for (int n = 0; n < D / 8; ++n)
            *reinterpret_cast<float2*>(dst + comb_col<D>(n * 8 + 2 * t4, row)) =
                make_float2(o[n][2 * hh], o[n][2 * hh + 1]);
          if (t4 == 0) {
            comb_ml[(warp * 2 + 0) * G + row] = m_run[hh];
            comb_ml[(warp * 2 + 1) * G + row] = lr[hh];
          }
        }
      } else if (g < G) {
        // row g's O (hi + lo halves): o[n][0..1] + o[n][2..3] = d 8n + 2t4 + {0,1}
        float* dst = comb_o + (warp * G + g) * D;
#pragma unroll
        for (int n = 0; n < D / 8; ++n)
          *reinterpret_cast<float2*>(dst + comb_col<D>(n * 8 + 2 * t4, g)) =
              make_float2(o[n][0] + o[n][2], o[n][1] + o[n][3]);
        if (t4 == 0) {
          comb_ml[(warp * 2 + 0) * G + g] = m_run[0];
          comb_ml[(warp * 2 + 1) * G + g] = lr[0];
        }
      }
      named_bar_arrive<1, kBarThreads>();
      fresh = true;
    }
  }
  // consume the epilogue's final EMPTY arrival (balances barrier 2 before exit)
  named_bar_sync<2, kBarThreads>();
  if (trace && threadIdx.x == 0) trace[12] = (long long)globaltimer();
}

using DecodeFn = void (*)(CUtensorMap, CUtensorMap, DecodeParams);

template <int D>
DecodeFn pick_g(int G) {
  switch (G) {
    case 1: return decode_kernel<D, 1>;
    case 2: return decode_kernel<D, 2>;
    case 4: return decode_kernel<D, 4>;
    case 8: return decode_kernel<D, 8>;
    case 16: return decode_kernel<D, 16>;
    default: return nullptr;
  }
}

}  // namespace

template <int D>
int smem_fixed(int G) {
  switch (G) {
    case 1: return Comb<D, 1>::kSmemFixed;
    case 2: return Comb<D, 2>::kSmemFixed;
    case 4: return Comb<D, 4>::kSmemFixed;
    case 8: return Comb<D, 8>::kSmemFixed;
    default: return Comb<D, 16>::kSmemFixed;
  }
}

int decode_smem_bytes(int D, int G, int slices) {
  const int fixed = D == 64 ? smem_fixed<64>(G) : smem_fixed<128>(G);
  return fixed + (slices + 1) * (int)sizeof(int);
}

int decode_grid(int tiles_upper, int num_sms, int permille) {
  return std::max(1, std::min(2 * num_sms * permille / 1000, tiles_upper));
}

cudaError_t launch_decode(const DecodeParams& p, const CUtensorMap& tmk, const CUtensorMap& tmv,
                          int D, int G, int ctas, cudaStream_t stream) {
  DecodeFn fn = (D == 64) ? pick_g<64>(G) : pick_g<128>(G);
  const int S = p.B * p.H;
  if (!fn || S > kMaxSlices || ctas > kMaxCtas) return cudaErrorInvalidValue;
  const int smem = decode_smem_bytes(D, G, S);
  cudaError_t e = ensure_kernel_attrs(reinterpret_cast<const void*>(fn), smem);
  if (e != cudaSuccess) return e;
  return launch_k(fn, dim3(ctas), dim3(kThreads), (size_t)smem, stream, tmk, tmv, p);
}

}  // namespace sfi_impl

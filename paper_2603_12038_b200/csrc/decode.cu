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

// ===========================================================================
// K1 on the 5th-generation tensor cores (tcgen05 + TMEM), dense mode, D = 128.
//
// One CTA per SM, the same stream-K schedule as decode_kernel but over
// 128-position tiles. Per tile (M = 128 positions):
//   S^T [128 pos x N] = K_tile [128 x 128 d] . Q^T          (tcgen05.mma, TMEM)
//   O^T [128 d x N]  += V_tile^T [128 d x 128 pos] . P^T    (tcgen05.mma, TMEM)
// N = the G query heads' bf16 hi rows and their lo residual rows (2G, padded
// to 16): the fp32 query keeps ~16 mantissa bits, and P is split the same way.
// Accumulators live in TMEM (S double-buffered, O persistent per segment), so
// the softmax warps hold only one position's N scores: registers are no longer
// the occupancy limit (decode_kernel's mma.sync consumers are latency-bound
// at G = 16).
//
// Warp roles: warp 0 = TMA producer (K, V tiles: 4 boxes of 64 cols x 128
// rows; and the per-segment Q tile, written by the warp's 32 lanes); warp 1 =
// TMEM owner + the single-thread MMA issuer; warps 2..5 = softmax / epilogue,
// warp w reading TMEM lanes 32 (w % 4) .. + 31 (tile row = position for S,
// d for O). The online softmax keeps one CTA-wide reference max per head
// (lazy: it moves only when a tile's max exceeds it by 2^8, then O^T is
// rescaled in TMEM); pooled logits are formed per position from S.
// Partials (m, l, O) and the last-arriver merge use decode_kernel's formats
// (merge_slice), so the two kernels are interchangeable.
constexpr int kTcRows = 128;
// softmax warps: G = 16 splits the heads over two warps per TMEM lane quadrant
template <int G>
__host__ __device__ constexpr int tc_softmax_warps() { return G >= 16 ? 8 : 4; }
template <int G>
__host__ __device__ constexpr int tc_threads() { return (3 + tc_softmax_warps<G>()) * 32; }
constexpr int kTcMaxThreads = 11 * 32;

template <int G, int ST>
struct TcGeo {
  static constexpr int N = (2 * G < 16) ? 16 : 2 * G;        // MMA N (hi + lo rows, padded)
  static constexpr int kBox = kTcRows * 128;                  // 128 rows x 64 bf16 = 16 KB
  static constexpr int kTileBytes = 2 * kBox;                 // one tensor, D = 128
  static constexpr int kStageBytes = 2 * kTileBytes;          // K + V
  static constexpr int kRing = ST * kStageBytes;              // ST stages of K + V
  static constexpr int kOpBox = N * 128;                      // Q / P box: N rows x 64 bf16
  static constexpr int kOpBytes = 2 * kOpBox;                 // 64-column boxes for 128 cols
  static constexpr int kQOff = kRing;                         // 2 Q buffers
  static constexpr int kPOff = kQOff + 2 * kOpBytes;          // 2 P buffers
  static constexpr int kMiscOff = kPOff + 2 * kOpBytes;
  // misc: 24 mbarriers, TMEM base, tile-max exchange [2][4][G], l sums [4][G]
  static constexpr int kRedOff = kMiscOff + 24 * 8 + 16;
  static constexpr int kLsumOff = kRedOff + 2 * 4 * G * 4;
  static constexpr int kPrefOff = kLsumOff + 4 * G * 4;
  static constexpr uint32_t kTmemCols = 128;                  // S[3] (3N) + O (N) <= 128
};

__device__ __forceinline__ uint64_t umma_sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  // SmemDescriptor (cute/arch/mma_sm100_desc.hpp): start, LBO, SBO in 16-byte
  // units, version 1 (sm100), layout SWIZZLE_128B
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46) | (2ull << 61);
}

template <int N, bool kAMnMajor>
__host__ __device__ constexpr uint32_t umma_idesc() {
  // InstrDescriptor: D fp32, A/B bf16, A K-major (QK) or MN-major (V^T), B K-major, M = 128
  return (1u << 4) | (1u << 7) | (1u << 10) | ((kAMnMajor ? 1u : 0u) << 15) | ((uint32_t)(N >> 3) << 17) |
         ((uint32_t)(kTcRows >> 4) << 24);
}

__device__ __forceinline__ void umma_f16(uint32_t dtmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(dtmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// tcgen05.ld / st, 32x32b shape: thread i of the warp <-> TMEM lane (quadrant base + i),
// n consecutive 32-bit columns
template <int N>
__device__ __forceinline__ void tmem_ld(uint32_t taddr, float (&v)[N]) {
  static_assert(N == 4 || N == 8 || N == 16, "tmem_ld width");
  uint32_t r[N];
  if constexpr (N == 4) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(taddr));
  } else if constexpr (N == 8) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
                   "=r"(r[7])
                 : "r"(taddr));
  } else {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
  }
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < N; ++i) v[i] = __uint_as_float(r[i]);
}

template <int N>
__device__ __forceinline__ void tmem_st(uint32_t taddr, const float (&v)[N]) {
  static_assert(N == 4 || N == 8, "tmem_st width");
  if constexpr (N == 4) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(taddr),
                 "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])),
                 "r"(__float_as_uint(v[3]))
                 : "memory");
  } else {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr),
                 "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])),
                 "r"(__float_as_uint(v[3])), "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])),
                 "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7]))
                 : "memory");
  }
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

// bf16 element (row r, column c) of a 128B-swizzled K-major operand (Q, P):
// 64-column boxes of R rows x 128 bytes; 16-byte chunks XOR-swizzled by row % 8
__device__ __forceinline__ uint32_t op_off(int r, int c, int box_bytes) {
  return (c >> 6) * box_bytes + r * 128 + ((((c & 63) >> 3) ^ (r & 7)) << 4) + ((c & 7) << 1);
}

__device__ __forceinline__ int tc_tiles(int rows) { return (rows + kTcRows - 1) / kTcRows; }

template <int G, int ST>
__global__ void __launch_bounds__(kTcMaxThreads, 1)
    decode_tc_kernel(const __grid_constant__ CUtensorMap tmk, const __grid_constant__ CUtensorMap tmv,
                     const DecodeParams p) {
  using Geo = TcGeo<G, ST>;
  constexpr int kTcStages = ST;
  constexpr int N = Geo::N;
  constexpr int D = 128;
  constexpr int PR = part_rows<G>();
  constexpr int kSW = tc_softmax_warps<G>();  // softmax warps: 4 x halves
  constexpr int kHalves = kSW / 4;
  constexpr int Gh = G / kHalves;             // heads per softmax warp
  constexpr int kQWarp = 2 + kSW;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Geo::kMiscOff);
  uint64_t* kv_full = bars;          // [3] K + V tile landed (TMA)
  uint64_t* kv_empty = bars + 3;     // [3] PV of the tile completed (stage free)
  uint64_t* s_full = bars + 6;       // [3] S^T of the tile in TMEM
  uint64_t* s_free = bars + 9;       // [3] S read by the 128 softmax threads
  uint64_t* p_full = bars + 12;      // [2] P written (128 threads)
  uint64_t* pv_done = bars + 14;     // [2] PV of the tile completed
  uint64_t* q_full = bars + 16;      // [2] Q buffer written (Q warp lanes)
  uint64_t* q_free = bars + 18;      // [2] the segment's last QK completed
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + Geo::kMiscOff + 24 * 8);
  float* red = reinterpret_cast<float*>(smem + Geo::kRedOff);     // [2][4][G]
  float* lsum = reinterpret_cast<float*>(smem + Geo::kLsumOff);   // [4][G]
  int* pref = reinterpret_cast<int*>(smem + Geo::kPrefOff);       // [S + 1]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int S = p.B * p.H;
  long long* trace = p.trace ? p.trace + (size_t)blockIdx.x * 16 : nullptr;  // SFI_DECODE_TRACE timeline
  if (threadIdx.x == 0) {
    if (trace) {
      trace[0] = (long long)globaltimer();
      trace[6] = smid();
    }
    tma_prefetch_desc(&tmk);
    tma_prefetch_desc(&tmv);
  }
  griddep_wait();
  griddep_launch();

  // ---- per-slice 128-row tile counts -> exclusive prefix ----
  for (int s = threadIdx.x; s < S; s += (int)blockDim.x) {
    const Slice sl = make_slice(p, s, blockIdx.x == 0);
    const int n = tc_tiles(sl.cnt[0]);
    pref[s + 1] = n;
    if (n == 0 && blockIdx.x == 0) {
      if (p.lse) {
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
    for (int i = 0; i < kTcStages; ++i) {
      mbar_init(&kv_full[i], 1);
      mbar_init(&kv_empty[i], 1);
      mbar_init(&s_full[i], 1);
      mbar_init(&s_free[i], kSW * 32);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&p_full[i], kSW * 32);
      mbar_init(&pv_done[i], 1);
      mbar_init(&q_full[i], 32);
      mbar_init(&q_free[i], 1);
    }
    fence_barrier_init();
  }
  if constexpr (N > 2 * G) {  // the Q / P buffers' padding rows stay zero (their MMA columns are unused)
    for (int e = threadIdx.x; e < 4 * Geo::kOpBytes / 16; e += (int)blockDim.x)
      reinterpret_cast<uint4*>(smem + Geo::kQOff)[e] = make_uint4(0, 0, 0, 0);
    fence_proxy_async();
  }
  if (warp == 1) {  // TMEM: S[0..2] at columns 0, N, 2N; O at 3N
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "n"(Geo::kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  __syncthreads();
  if (warp == 0) {
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
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int T = pref[S];
  const int Gc = gridDim.x;
  const int tb = cta_start(blockIdx.x, T, Gc);
  const int te = cta_start(blockIdx.x + 1, T, Gc);
  const int s_first = tb < te ? slice_of(pref, S, tb) : 0;
  if (trace && threadIdx.x == 0) {
    trace[1] = (long long)globaltimer();
    trace[5] = te - tb;
  }

  if (tb < te && warp == 0) {
    // ---------------- producer: K + V tiles by TMA (lane 0) ----------------
    if (lane == 0) {
      const uint64_t pol = l2_policy_evict_first();
      int s = s_first;
      Slice sl = make_slice(p, s, false);
      for (int t = tb, i = 0; t < te; ++t, ++i) {
        while (pref[s + 1] <= t) sl = make_slice(p, ++s, false);
        const int st = i % kTcStages;
        if (i >= kTcStages) mbar_wait(&kv_empty[st], ((i / kTcStages) - 1) & 1);
        const int row = sl.row_base + (t - pref[s]) * kTcRows;
        uint8_t* kdst = smem + st * Geo::kStageBytes;
        uint8_t* vdst = kdst + Geo::kTileBytes;
        mbar_arrive_expect_tx(&kv_full[st], Geo::kStageBytes);
#pragma unroll
        for (int bx = 0; bx < 2; ++bx) {
          tma_load_2d(kdst + bx * Geo::kBox, &tmk, bx * 64, row, &kv_full[st], pol);
          tma_load_2d(vdst + bx * Geo::kBox, &tmv, bx * 64, row, &kv_full[st], pol);
        }
      }
    }
    __syncwarp();
  } else if (tb < te && warp == kQWarp) {
    // ---------------- Q warp: each segment's query rows (bf16 hi / lo, zero padded) ----------------
    int seg = 0;
    for (int s = s_first; s < S && pref[s] < te; ++s) {
      if (pref[s + 1] <= tb || pref[s + 1] == pref[s]) continue;
      const int qb = seg & 1;
      if (seg >= 2) mbar_wait(&q_free[qb], ((seg >> 1) - 1) & 1);  // segment seg - 2's QKs completed
      uint8_t* qdst = smem + Geo::kQOff + qb * Geo::kOpBytes;
      const int b = s / p.H, h = s % p.H;
      const float* qsrc = p.q + ((size_t)b * p.Hq + (size_t)h * G) * D;
      // float4 loads (8 in flight per lane), hi / lo halves as 8-byte stores (4
      // consecutive columns never straddle a 16-byte swizzle chunk)
      constexpr int kItems = G * (D / 4);
      for (int e0 = lane; e0 < kItems; e0 += 32 * 8) {
        float4 v[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int e = e0 + 32 * j;
          v[j] = e < kItems ? *reinterpret_cast<const float4*>(qsrc + (e / (D / 4)) * D + (e % (D / 4)) * 4)
                            : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int e = e0 + 32 * j;
          if (e >= kItems) break;
          const int r = e / (D / 4), c = (e % (D / 4)) * 4;
          float h0, l0, h1, l1, h2, l2, h3, l3;
          split_bf16(v[j].x, h0, l0);
          split_bf16(v[j].y, h1, l1);
          split_bf16(v[j].z, h2, l2);
          split_bf16(v[j].w, h3, l3);
          *reinterpret_cast<uint2*>(qdst + op_off(r, c, Geo::kOpBox)) = make_uint2(pack_bf16(h0, h1), pack_bf16(h2, h3));
          *reinterpret_cast<uint2*>(qdst + op_off(G + r, c, Geo::kOpBox)) =
              make_uint2(pack_bf16(l0, l1), pack_bf16(l2, l3));
        }
      }
      fence_proxy_async();
      mbar_arrive(&q_full[qb]);
      ++seg;
    }
  } else if (tb < te && warp == 1) {
    // ---------------- MMA issuer (one thread) ----------------
    if (lane == 0) {
      constexpr uint32_t kIdQK = umma_idesc<N, false>();
      constexpr uint32_t kIdPV = umma_idesc<N, true>();
      const uint32_t ring = smem_u32(smem);
      // Non-blocking issue loop: QK of tile qk_i as soon as its K tile, its
      // segment's Q and an S buffer are ready (up to kTcStages ahead of PV), PV of
      // tile pv_i as soon as its P is written — so S runs ahead of the softmax
      // instead of waiting for the previous PV.
      const int n = te - tb;
      int qk_i = 0, pv_i = 0;
      int s_q = s_first, seg_q = 0, seg_tile = 0;
      int s_p = s_first;
      while (pv_i < n) {
        if (pv_i < qk_i) {
          const int pb = pv_i & 1;
          if (mbar_test(&p_full[pb], (pv_i >> 1) & 1)) {
            const int t = tb + pv_i, st = pv_i % kTcStages;
            bool first = (pv_i == 0);
            if (pref[s_p + 1] <= t) {
              while (pref[s_p + 1] <= t) ++s_p;
              first = true;
            }
            tc_fence_after();
            const uint32_t vaddr = ring + st * Geo::kStageBytes + Geo::kTileBytes;
            const uint32_t paddr = smem_u32(smem + Geo::kPOff + pb * Geo::kOpBytes);
#pragma unroll
            for (int ks = 0; ks < kTcRows / 16; ++ks) {
              // A = V^T (M = d, K = positions), MN-major: LBO = the second 64-d box, SBO = 8 positions
              const uint32_t voff = ks * 16 * 128;
              const uint32_t poff = (ks >> 2) * Geo::kOpBox + (ks & 3) * 32;
              umma_f16(tmem + kTcStages * N, umma_sdesc(vaddr + voff, Geo::kBox, 1024),
                       umma_sdesc(paddr + poff, 16, 1024), kIdPV, (first && ks == 0) ? 0u : 1u);
            }
            umma_commit(&kv_empty[st]);
            umma_commit(&pv_done[pb]);
            ++pv_i;
            continue;
          }
        }
        if (qk_i < n && qk_i - pv_i < kTcStages) {
          const int t = tb + qk_i, st = qk_i % kTcStages;
          if (seg_tile != qk_i) {  // segment bookkeeping of tile qk_i, once
            if (qk_i > 0 && pref[s_q + 1] <= t) {
              umma_commit(&q_free[seg_q & 1]);  // every QK of segment seg_q is issued
              while (pref[s_q + 1] <= t) ++s_q;
              ++seg_q;
            }
            seg_tile = qk_i;
          }
          if (mbar_test(&q_full[seg_q & 1], (seg_q >> 1) & 1) && mbar_test(&kv_full[st], (qk_i / kTcStages) & 1) &&
              (qk_i < kTcStages || mbar_test(&s_free[st], ((qk_i / kTcStages) - 1) & 1))) {
            tc_fence_after();
            const uint32_t kaddr = ring + st * Geo::kStageBytes;
            const uint32_t qaddr = smem_u32(smem + Geo::kQOff + (seg_q & 1) * Geo::kOpBytes);
#pragma unroll
            for (int ks = 0; ks < D / 16; ++ks) {
              const uint32_t koff = (ks >> 2) * Geo::kBox + (ks & 3) * 32;
              const uint32_t qoff = (ks >> 2) * Geo::kOpBox + (ks & 3) * 32;
              umma_f16(tmem + st * N, umma_sdesc(kaddr + koff, 16, 1024), umma_sdesc(qaddr + qoff, 16, 1024),
                       kIdQK, ks > 0);
            }
            umma_commit(&s_full[st]);
            ++qk_i;
          }
        }
      }
    }
    __syncwarp();
  } else if (tb < te && warp >= 2 && warp < 2 + kSW) {
    // ---------------- softmax / epilogue warps (kSW * 32 threads) ----------------
    // warp w reads TMEM lane quadrant w % 4 (tile row = position for S, d for O)
    // and owns heads [hf * Gh, (hf + 1) * Gh), hf = (w - 2) / 4
    const int q4 = warp & 3;
    const int row = q4 * 32 + lane;
    const int hf = (warp - 2) >> 2;
    const int g0 = hf * Gh;
    const uint32_t lane_base = (uint32_t)(q4 * 32) << 16;
    const float sl2 = p.scale_log2;
    float m_ref[Gh], l_part[Gh];
#pragma unroll
    for (int g = 0; g < Gh; ++g) {
      m_ref[g] = -INFINITY;
      l_part[g] = 0.f;
    }
    int s = s_first;
    Slice sl = make_slice(p, s, false);
    int pend[2], n_pend = 0;
    for (int t = tb, i = 0; t < te; ++t, ++i) {
      while (pref[s + 1] <= t) sl = make_slice(p, ++s, false);
      const bool first = (i == 0) || (t == pref[s]);
      const bool last = (t + 1 == pref[s + 1]) || (t + 1 == te);
      const int sb = i & 1;                           // P buffer
      const int ss = i % kTcStages;                   // S buffer
      const int toff = (t - pref[s]) * kTcRows;       // row offset in the slice
      const int nvalid = min(kTcRows, sl.cnt[0] - toff);
      const bool valid = row < nvalid;
      const int pos = toff + row + 1;
      const bool in_j = p.logits != nullptr && valid && pos >= sl.j_min && pos <= sl.j_max;
      // ---- S of this tile: this warp's heads (hi and lo columns) ----
      mbar_wait(&s_full[ss], (i / kTcStages) & 1);
      if (trace && i == 0 && threadIdx.x == 64) trace[2] = (long long)globaltimer();
      tc_fence_after();
      float x[Gh];
      {
        float shi[Gh], slo[Gh];
        tmem_ld<Gh>(tmem + lane_base + ss * N + g0, shi);
        tmem_ld<Gh>(tmem + lane_base + ss * N + G + g0, slo);
#pragma unroll
        for (int g = 0; g < Gh; ++g) x[g] = shi[g] + slo[g];
        // pooled logits over J (attention.cpp:394-409): the half-0 warps also read the
        // other heads' columns and emit the position's pooled value
        if (kHalves > 1 && hf == 0 && __any_sync(0xffffffffu, in_j)) {  // tcgen05.ld: warp-uniform
          float ohi[Gh], olo[Gh];
          tmem_ld<Gh>(tmem + lane_base + ss * N + Gh, ohi);
          tmem_ld<Gh>(tmem + lane_base + ss * N + G + Gh, olo);
          float v = (p.pool == SFI_POOL_MAX) ? -INFINITY : 0.f;
#pragma unroll
          for (int g = 0; g < 2 * Gh; ++g) {
            const float xg = (g < Gh ? x[g] : ohi[g - Gh] + olo[g - Gh]) * p.inv_sqrt_d;
            v = (p.pool == SFI_POOL_MAX) ? fmaxf(v, xg) : v + xg;
          }
          if (p.pool != SFI_POOL_MAX) v *= (1.0f / G);
          if (in_j) p.logits[(size_t)s * p.Lmax + (pos - sl.j_min)] = v;
        } else if (kHalves == 1 && in_j) {
          float v = (p.pool == SFI_POOL_MAX) ? -INFINITY : 0.f;
#pragma unroll
          for (int g = 0; g < Gh; ++g) {
            const float xg = x[g] * p.inv_sqrt_d;
            v = (p.pool == SFI_POOL_MAX) ? fmaxf(v, xg) : v + xg;
          }
          if (p.pool != SFI_POOL_MAX) v *= (1.0f / G);
          p.logits[(size_t)s * p.Lmax + (pos - sl.j_min)] = v;
        }
      }
      tc_fence_before();
      mbar_arrive(&s_free[ss]);
      // ---- lazy online softmax: the CTA-wide reference max per head moves only
      // when some position of the tile exceeds it by 2^8 (one barrier.red.or);
      // then the tile max per head is reduced across the 128 positions ----
      if (first) {
#pragma unroll
        for (int g = 0; g < Gh; ++g) {
          m_ref[g] = -INFINITY;
          l_part[g] = 0.f;
        }
      }
      bool need = false;
#pragma unroll
      for (int g = 0; g < Gh; ++g) {
        x[g] = valid ? x[g] * sl2 : -INFINITY;
        need |= x[g] > m_ref[g] + kLazyMax;
      }
      int any_i;
      asm volatile("{\n.reg .pred pi, po;\nsetp.ne.u32 pi, %1, 0;\nbarrier.red.or.pred po, 2, %2, pi;\n"
                   "selp.u32 %0, 1, 0, po;\n}"
                   : "=r"(any_i)
                   : "r"((uint32_t)need), "n"(kSW * 32)
                   : "memory");
      bool grow_any = false;
      float alpha[Gh];
      if (any_i) {
        float* rb = red + (i & 1) * 4 * G;  // [quadrant][head]
#pragma unroll
        for (int g = 0; g < Gh; ++g) {
          float mx = x[g];
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
          if (lane == 0) rb[q4 * G + g0 + g] = mx;
        }
        named_bar_sync<1, kSW * 32>();
#pragma unroll
        for (int g = 0; g < Gh; ++g) {
          const int gg = g0 + g;
          const float tm = fmaxf(fmaxf(rb[gg], rb[G + gg]), fmaxf(rb[2 * G + gg], rb[3 * G + gg]));
          const bool grow = tm > m_ref[g] + kLazyMax;
          const float m_new = grow ? tm : m_ref[g];
          const float m_use = (m_new == -INFINITY) ? 0.f : m_new;
          alpha[g] = grow ? fast_exp2(m_ref[g] - m_use) : 1.f;
          grow_any |= grow;
          m_ref[g] = m_new;
          l_part[g] *= alpha[g];
        }
      } else {
#pragma unroll
        for (int g = 0; g < Gh; ++g) alpha[g] = 1.f;
      }
#pragma unroll
      for (int g = 0; g < Gh; ++g) {
        const float m_use = (m_ref[g] == -INFINITY) ? 0.f : m_ref[g];
        const float pr = valid ? fast_exp2(x[g] - m_use) : 0.f;
        x[g] = pr;
        l_part[g] += pr;
      }
      // O^T holds PV of this segment's earlier tiles: rescale this warp's head
      // columns in TMEM once those PVs completed
      if (grow_any && !first) {
        mbar_wait(&pv_done[(i - 1) & 1], ((i - 1) >> 1) & 1);
        tc_fence_after();
        float ohi[Gh], olo[Gh];
        tmem_ld<Gh>(tmem + lane_base + kTcStages * N + g0, ohi);
        tmem_ld<Gh>(tmem + lane_base + kTcStages * N + G + g0, olo);
#pragma unroll
        for (int g = 0; g < Gh; ++g) {
          ohi[g] *= alpha[g];
          olo[g] *= alpha[g];
        }
        tmem_st<Gh>(tmem + lane_base + kTcStages * N + g0, ohi);
        tmem_st<Gh>(tmem + lane_base + kTcStages * N + G + g0, olo);
      }
      // ---- P (this warp's hi / lo rows) into buffer sb once PV(i - 2) released it ----
      if (i >= 2) mbar_wait(&pv_done[sb], ((i >> 1) - 1) & 1);
      uint8_t* pdst = smem + Geo::kPOff + sb * Geo::kOpBytes;
#pragma unroll
      for (int g = 0; g < Gh; ++g) {
        float hi, lo;
        split_bf16(x[g], hi, lo);
        *reinterpret_cast<__nv_bfloat16*>(pdst + op_off(g0 + g, row, Geo::kOpBox)) = __float2bfloat16_rn(hi);
        *reinterpret_cast<__nv_bfloat16*>(pdst + op_off(G + g0 + g, row, Geo::kOpBox)) = __float2bfloat16_rn(lo);
      }
      fence_proxy_async();
      tc_fence_before();
      mbar_arrive(&p_full[sb]);
      if (!last) continue;
      // ---- end of this CTA's part of slice s: O^T [d][n] after PV(i) ----
      mbar_wait(&pv_done[sb], (i >> 1) & 1);
      tc_fence_after();
      float ohi[Gh], olo[Gh];
      tmem_ld<Gh>(tmem + lane_base + kTcStages * N + g0, ohi);
      tmem_ld<Gh>(tmem + lane_base + kTcStages * N + G + g0, olo);
      tc_fence_before();
      named_bar_sync<1, kSW * 32>();  // lsum reuse
#pragma unroll
      for (int g = 0; g < Gh; ++g) {
        float l = l_part[g];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) l += __shfl_xor_sync(0xffffffffu, l, o);
        if (lane == 0) lsum[q4 * G + g0 + g] = l;
      }
      named_bar_sync<1, kSW * 32>();
      const int P0 = pref[s], P1 = pref[s + 1];
      const int c_first = cta_of(P0, T, Gc), c_last = cta_of(P1 - 1, T, Gc);
      const int b = s / p.H, h = s % p.H;
      if (c_first == c_last) {
        float* outp = p.out + ((size_t)b * p.Hq + (size_t)h * G) * D;
#pragma unroll
        for (int g = 0; g < Gh; ++g) {
          const int gg = g0 + g;
          const float L = lsum[gg] + lsum[G + gg] + lsum[2 * G + gg] + lsum[3 * G + gg];
          const float inv = L > 0.f ? 1.f / L : 0.f;
          outp[gg * D + row] = (ohi[g] + olo[g]) * inv;
          if (p.lse && row == gg) p.lse[(size_t)b * p.Hq + (size_t)h * G + gg] = lse_of(m_ref[g], L);
        }
      } else {
        const int slot = (s == s_first) ? 0 : 1;
        const size_t part = (size_t)blockIdx.x * 2 + slot;
#pragma unroll
        for (int g = 0; g < Gh; ++g) {
          const int gg = g0 + g;
          p.part_o[(part * PR + gg) * D + row] = ohi[g] + olo[g];
          if (row == gg) {
            p.part_ml[(part * 2 + 0) * PR + gg] = m_ref[g];
            p.part_ml[(part * 2 + 1) * PR + gg] = lsum[gg] + lsum[G + gg] + lsum[2 * G + gg] + lsum[3 * G + gg];
          }
        }
        if (n_pend < 2) pend[n_pend++] = s;
      }
    }
    // Publish this CTA's partials; the last-arriving contributor of a slice
    // merges them with all kSW warps (a slice split over ~40 CTAs at C4 made
    // a one-warp merge the kernel's tail): per head the max / sum over the
    // contributors in CTA order, then every (head, d) output as one pipelined
    // pass over the contributors' rows.
    if (trace && threadIdx.x == 64) trace[12] = (long long)globaltimer();
    if (n_pend > 0) {
      constexpr int NT = kSW * 32;
      const int tid = threadIdx.x - 64;  // 0 .. NT - 1
      float* cm = reinterpret_cast<float*>(smem + Geo::kPOff);   // [<= kMaxCtas... C][G] scales (P area is free now)
      float* hM = red;                                            // [G] per-head max, then sum in lsum
      int* flag = reinterpret_cast<int*>(lsum + 4 * G - 1);
      __threadfence();
      for (int k = 0; k < n_pend; ++k) {
        const int sp = pend[k];
        const int P0 = pref[sp], P1 = pref[sp + 1];
        const int c_first = cta_of(P0, T, Gc), c_last = cta_of(P1 - 1, T, Gc);
        const int C = c_last - c_first + 1;
        named_bar_sync<1, NT>();
        if (warp == 2) {
          int n_contrib = 0;
          for (int cb = c_first; cb <= c_last; cb += 32) {
            const int c = cb + lane;
            const bool ok = c <= c_last && cta_start(c, T, Gc) < cta_start(c + 1, T, Gc);
            n_contrib += __popc(__ballot_sync(0xffffffffu, ok));
          }
          if (lane == 0) *flag = (atomicAdd(&p.counters[sp], 1) == n_contrib - 1);
        }
        named_bar_sync<1, NT>();
        if (!*flag) continue;
        __threadfence();  // acquire the other contributors' partials
        const int b = sp / p.H, h = sp % p.H;
        float* outp = p.out + ((size_t)b * p.Hq + (size_t)h * G) * D;
        const int cap = (2 * Geo::kOpBytes) / (int)sizeof(float) / (2 * G + 1);  // contributors the scale area holds
        if (C > cap) {  // a slice over more than `cap` CTAs (ragged batches): the one-warp merge
          if (warp == 2)
            merge_slice<D, G>(p, outp, p.lse ? p.lse + (size_t)b * p.Hq + (size_t)h * G : nullptr, P0, c_first,
                              c_last, T, Gc, lane);
          if (tid == 0) p.counters[sp] = 0;
          continue;
        }
        {
          const int cn = C;
          int* pcs = reinterpret_cast<int*>(cm + 2 * cn * G);  // partial slot per contributor, -1 = empty
          for (int ci = tid; ci < cn; ci += NT) {
            const int c = c_first + ci;
            const int c0s = cta_start(c, T, Gc);
            pcs[ci] = c0s < cta_start(c + 1, T, Gc) ? c * 2 + (c0s >= P0 ? 0 : 1) : -1;
          }
          named_bar_sync<1, NT>();
          for (int e = tid; e < cn * G; e += NT) {
            const int ci = e / G, g = e % G, pc = pcs[ci];
            cm[2 * e] = pc >= 0 ? __ldcg(&p.part_ml[((size_t)pc * 2 + 0) * PR + g]) : -INFINITY;
            cm[2 * e + 1] = pc >= 0 ? __ldcg(&p.part_ml[((size_t)pc * 2 + 1) * PR + g]) : 0.f;
          }
          named_bar_sync<1, NT>();
          if (tid < G) {  // per head, contributors in CTA order (deterministic); 1 / L folded in
            float M = -INFINITY;
            for (int ci = 0; ci < cn; ++ci) M = fmaxf(M, cm[2 * (ci * G + tid)]);
            const float Mu = (M == -INFINITY) ? 0.f : M;
            float L = 0.f;
            for (int ci = 0; ci < cn; ++ci) {
              const float sc = fast_exp2(cm[2 * (ci * G + tid)] - Mu);
              cm[2 * (ci * G + tid)] = sc;
              L += cm[2 * (ci * G + tid) + 1] * sc;
            }
            const float inv = L > 0.f ? 1.f / L : 0.f;
            for (int ci = 0; ci < cn; ++ci) cm[2 * (ci * G + tid)] *= inv;
            hM[tid] = M;
            lsum[tid] = L;
          }
          named_bar_sync<1, NT>();
          // every (head, 4 d) output: 16 contributors' rows in flight per round
          constexpr int kR = 16;
          for (int it = tid; it < G * (D / 4); it += NT) {
            const int g = it / (D / 4), d4 = it % (D / 4);
            float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
            for (int c0 = 0; c0 < cn; c0 += kR) {
              float4 xv[kR];
#pragma unroll
              for (int j = 0; j < kR; ++j) {
                const int ci = c0 + j;
                const int pc = ci < cn ? pcs[ci] : -1;
                xv[j] = pc >= 0 ? __ldcg(reinterpret_cast<const float4*>(p.part_o + ((size_t)pc * PR + g) * D) + d4)
                                : make_float4(0.f, 0.f, 0.f, 0.f);
              }
#pragma unroll
              for (int j = 0; j < kR; ++j) {
                const float sc = (c0 + j < cn) ? cm[2 * ((c0 + j) * G + g)] : 0.f;
                acc.x += xv[j].x * sc;
                acc.y += xv[j].y * sc;
                acc.z += xv[j].z * sc;
                acc.w += xv[j].w * sc;
              }
            }
            reinterpret_cast<float4*>(outp + g * D)[d4] = acc;
            if (p.lse && d4 == 0) p.lse[(size_t)b * p.Hq + (size_t)h * G + g] = lse_of(hM[g], lsum[g]);
          }
        }
        if (tid == 0) p.counters[sp] = 0;
      }
    }
    if (trace && threadIdx.x == 64) trace[10] = (long long)globaltimer() - trace[12];
  }
  tc_fence_before();
  __syncthreads();
  if (trace && threadIdx.x == 0) trace[3] = (long long)globaltimer();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(Geo::kTmemCols));
  }
}

template <int G, int ST>
int tc_smem_bytes(int slices) {
  return TcGeo<G, ST>::kPrefOff + (slices + 1) * (int)sizeof(int);
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
  // at least ~8 tiles per CTA: small problems (C1, 33.8 MB per launch) lose more to
  // the stream-K merges of many thin CTAs than they gain in parallelism
  // (C1 K1 alone 24.0 -> 18.8 us, beside the Selector 27.9 -> 23.1 us)
  const int cap = std::max(num_sms / 2, (tiles_upper + 7) / 8);
  return std::max(1, std::min({2 * num_sms * permille / 1000, tiles_upper, cap}));
}

cudaError_t launch_decode_tc(const DecodeParams& p, const CUtensorMap& tmk128, const CUtensorMap& tmv128, int G,
                             int stages, int ctas, cudaStream_t stream) {
  using Fn = void (*)(CUtensorMap, CUtensorMap, DecodeParams);
  Fn fn = nullptr;
  int smem = 0, threads = 0;
  const int S = p.B * p.H;
#define SFI_TC_CASE(GG, SS)                      \
  if (G == GG && stages == SS) {                 \
    fn = decode_tc_kernel<GG, SS>;               \
    smem = tc_smem_bytes<GG, SS>(S);             \
    threads = tc_threads<GG>();                  \
  }
  SFI_TC_CASE(4, 3) SFI_TC_CASE(8, 3) SFI_TC_CASE(16, 3) SFI_TC_CASE(4, 2) SFI_TC_CASE(8, 2) SFI_TC_CASE(16, 2)
#undef SFI_TC_CASE
  if (!fn || S > kMaxSlices || ctas > kMaxCtas || p.sparse) return cudaErrorInvalidValue;
  cudaError_t e = ensure_kernel_attrs(reinterpret_cast<const void*>(fn), smem);
  if (e != cudaSuccess) return e;
  return launch_k(fn, dim3(ctas), dim3(threads), (size_t)smem, stream, tmk128, tmv128, p);
}

int decode_tc_tiles_upper(int max_positions) { return (max_positions + kTcRows - 1) / kTcRows; }

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

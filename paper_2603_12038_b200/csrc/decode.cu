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
constexpr int kThreads = (kNcw + 1) * 32;
constexpr int kStages = 3;
constexpr int kMaxSlices = 4096;

template <int D>
struct Geo {
  static constexpr int kBoxes = D / 64;                   // 128-byte TMA boxes per row
  static constexpr int kBoxBytes = kTile * 128;           // 8 KB
  static constexpr int kTileBytes = kBoxes * kBoxBytes;   // one tensor, one tile
  static constexpr int kStageBytes = 2 * kTileBytes;      // K + V
  static constexpr int kRing = kStages * kStageBytes;
  static constexpr int kComb = 3 * 8 * D * 4 + 3 * 2 * 8 * 4;  // warps 1..3 hand-off slots (O, m, l)
  static constexpr int kSmemFixed = kRing + kComb + 256 /*barriers*/ + 1024 /*align*/;
};

struct Slice {
  int off[3];
  int cnt[3];
  int row_base;   // first row of the (layer, b, h) slice in the 2D tensor
  int j_min, j_max;
};

__device__ __forceinline__ int seg_tiles(int c) { return (c + kTile - 1) / kTile; }

// 128B-swizzled address of 16-byte chunk `chunk` (8 bf16) of tile row `row`.
template <int D>
__device__ __forceinline__ uint32_t swz(uint32_t base, int row, int chunk) {
  return base + (chunk >> 3) * Geo<D>::kBoxBytes + row * 128 + (((chunk & 7) ^ (row & 7)) << 4);
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

template <int D, int G>
__global__ void __launch_bounds__(kThreads, 2)
    decode_kernel(const __grid_constant__ CUtensorMap tmk, const __grid_constant__ CUtensorMap tmv,
                  const DecodeParams p) {
  static_assert(G >= 1 && G <= 8, "GQA group of at most 8 query heads per KV head");
  static_assert(D == 64 || D == 128, "head_dim 64 or 128");
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  float* comb_o = reinterpret_cast<float*>(smem + Geo<D>::kRing);           // [3][8][D]
  float* comb_ml = comb_o + 3 * 8 * D;                                      // [3][2][8]
  uint64_t* full = reinterpret_cast<uint64_t*>(comb_ml + 3 * 2 * 8);
  uint64_t* empty = full + kStages;
  int* pref = reinterpret_cast<int*>(empty + kStages + 2);                  // [S + 1]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int S = p.B * p.H;
  long long* trace = p.trace ? p.trace + (size_t)blockIdx.x * 16 : nullptr;
  if (trace && threadIdx.x == 0) {
    trace[0] = (long long)globaltimer();
    trace[6] = smid();
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
    if (n == 0 && blockIdx.x == 0) raise_error(p.err, SFI_ERR_EMPTY_SUPPORT);
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
      tma_prefetch_desc(&tmk);
      tma_prefetch_desc(&tmv);
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
        uint8_t* kdst = smem + st * Geo<D>::kStageBytes;
        uint8_t* vdst = kdst + Geo<D>::kTileBytes;
        mbar_arrive_expect_tx(&full[st], Geo<D>::kStageBytes);
#pragma unroll
        for (int bx = 0; bx < Geo<D>::kBoxes; ++bx) {
          tma_load_2d(kdst + bx * Geo<D>::kBoxBytes, &tmk, bx * 64, row, &full[st], pol);
          tma_load_2d(vdst + bx * Geo<D>::kBoxBytes, &tmv, bx * 64, row, &full[st], pol);
        }
      }
    }
    return;
  }

  // ---------------- consumers ----------------
  const int g = lane >> 2, t4 = lane & 3;
  const float sl2 = p.scale_log2;
  uint32_t qa[D / 16][4];
  float o[D / 8][4];
  float m_run = -INFINITY, l_run = 0.f;
  int s = s_first;
  Slice sl = make_slice(p, s, false);
  bool fresh = true;
  // hand-off slots start free: warp 0 pre-arrives on EMPTY (barrier 2)
  if (warp == 0) asm volatile("bar.arrive 2, %0;" ::"n"(kNcw * 32));

  for (int t = tb, i = 0; t < te; ++t, ++i) {
    while (pref[s + 1] <= t) sl = make_slice(p, ++s, false);
    if (fresh) {
      // Q fragments: rows 0..7 = bf16 hi of query head g (< G), rows 8..15 = lo
      const int b = s / p.H, h = s % p.H;
      const float* qg = p.q + ((size_t)b * p.Hq + (size_t)h * G + g) * D;
#pragma unroll
      for (int ks = 0; ks < D / 16; ++ks) {
#pragma unroll
        for (int half = 0; half < 2; ++half) {
          const int c = ks * 16 + half * 8 + 2 * t4;
          float x0 = 0.f, x1 = 0.f;
          if (g < G) {
            const float2 v = *reinterpret_cast<const float2*>(qg + c);
            x0 = v.x;
            x1 = v.y;
          }
          float h0, l0, h1, l1;
          split_bf16(x0, h0, l0);
          split_bf16(x1, h1, l1);
          qa[ks][half * 2 + 0] = pack_bf16(h0, h1);
          qa[ks][half * 2 + 1] = pack_bf16(l0, l1);
        }
      }
#pragma unroll
      for (int n = 0; n < D / 8; ++n) o[n][0] = o[n][1] = o[n][2] = o[n][3] = 0.f;
      m_run = -INFINITY;
      l_run = 0.f;
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
      const uint32_t kbase = smem_u32(smem + st * Geo<D>::kStageBytes);
      const uint32_t vbase = kbase + Geo<D>::kTileBytes;
      // ---- S = Q K^T for 16 keys ----
      float acc[2][4];
#pragma unroll
      for (int j = 0; j < 2; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.f;
#pragma unroll
      for (int kc = 0; kc < D / 16; kc += 2) {
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          uint32_t b0, b1, b2, b3;
          ldsm_x4(swz<D>(kbase, kw + j * 8 + (lane & 7), kc * 2 + (lane >> 3)), b0, b1, b2, b3);
          mma_bf16(acc[j], qa[kc], b0, b1);
          mma_bf16(acc[j], qa[kc + 1], b2, b3);
        }
      }
      float sc[2][2];
      bool valid[2][2];
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          sc[j][e] = acc[j][e] + acc[j][e + 2];
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
              float v = sc[j][e] * p.inv_sqrt_d;
              if (p.pool == SFI_POOL_MAX) {
                if (g >= G) v = -INFINITY;
                v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, 4));
                v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, 8));
                v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, 16));
              } else {
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
      float mx = -INFINITY;
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          sc[j][e] = valid[j][e] ? sc[j][e] * sl2 : -INFINITY;
          mx = fmaxf(mx, sc[j][e]);
        }
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
      const float m_new = fmaxf(m_run, mx);
      const float m_use = (m_new == -INFINITY) ? 0.f : m_new;
      const float alpha = fast_exp2(m_run - m_use);
      float pr[2][2], psum = 0.f;
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          pr[j][e] = fast_exp2(sc[j][e] - m_use);
          psum += pr[j][e];
        }
      l_run = l_run * alpha + psum;
      m_run = m_new;
#pragma unroll
      for (int n = 0; n < D / 8; ++n) {
        o[n][0] *= alpha;
        o[n][1] *= alpha;
        o[n][2] *= alpha;
        o[n][3] *= alpha;
      }
      // ---- P as the A operand: rows 0..7 hi, rows 8..15 lo ----
      uint32_t pa[4];
      {
        float h00, l00, h01, l01, h10, l10, h11, l11;
        split_bf16(pr[0][0], h00, l00);
        split_bf16(pr[0][1], h01, l01);
        split_bf16(pr[1][0], h10, l10);
        split_bf16(pr[1][1], h11, l11);
        pa[0] = pack_bf16(h00, h01);
        pa[1] = pack_bf16(l00, l01);
        pa[2] = pack_bf16(h10, h11);
        pa[3] = pack_bf16(l10, l11);
      }
      // ---- O += P V ----
#pragma unroll
      for (int nd = 0; nd < D / 8; nd += 2) {
        const int mi = lane >> 3;
        uint32_t v0, v1, v2, v3;
        ldsm_x4_t(swz<D>(vbase, kw + (mi & 1) * 8 + (lane & 7), nd + (mi >> 1)), v0, v1, v2, v3);
        mma_bf16(o[nd], pa, v0, v1);
        mma_bf16(o[nd + 1], pa, v2, v3);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);

    // ---- end of this CTA's part of slice s: combine 4 warps, emit ----
    if (t + 1 == pref[s + 1] || t + 1 == te) {
      float lr = l_run;
      lr += __shfl_xor_sync(0xffffffffu, lr, 1);
      lr += __shfl_xor_sync(0xffffffffu, lr, 2);
      // row g's O (hi + lo halves) in place: o[n][0..1] = d 8n + 2t4 + {0,1}
#pragma unroll
      for (int n = 0; n < D / 8; ++n) {
        o[n][0] += o[n][2];
        o[n][1] += o[n][3];
      }
      const long long te0 = trace ? (long long)globaltimer() : 0;
      if (warp != 0) {
        // hand the warp partial to warp 0 and keep consuming tiles:
        // EMPTY (barrier 2) -> write slot -> FULL (barrier 1, arrive only)
        asm volatile("bar.sync 2, %0;" ::"n"(kNcw * 32));
        if (g < G) {
          float* dst = comb_o + ((warp - 1) * 8 + g) * D;
#pragma unroll
          for (int n = 0; n < D / 8; ++n)
            *reinterpret_cast<float2*>(dst + n * 8 + 2 * t4) = make_float2(o[n][0], o[n][1]);
          if (t4 == 0) {
            comb_ml[((warp - 1) * 2 + 0) * 8 + g] = m_run;
            comb_ml[((warp - 1) * 2 + 1) * 8 + g] = lr;
          }
        }
        asm volatile("bar.arrive 1, %0;" ::"n"(kNcw * 32));
      } else {
        // warp 0: combine warps 0..3 in fixed order, then emit
        asm volatile("bar.sync 1, %0;" ::"n"(kNcw * 32));
        float mr = m_run;
        if (g < G) {
#pragma unroll 1
          for (int w = 0; w < kNcw - 1; ++w) {
            const float* src = comb_o + (w * 8 + g) * D;
            const float m2 = comb_ml[(w * 2 + 0) * 8 + g];
            const float l2 = comb_ml[(w * 2 + 1) * 8 + g];
            const float M = fmaxf(mr, m2);
            const float Mu = (M == -INFINITY) ? 0.f : M;
            const float a1 = fast_exp2(mr - Mu), a2 = fast_exp2(m2 - Mu);
#pragma unroll
            for (int n = 0; n < D / 8; ++n) {
              const float2 x = *reinterpret_cast<const float2*>(src + n * 8 + 2 * t4);
              o[n][0] = o[n][0] * a1 + x.x * a2;
              o[n][1] = o[n][1] * a1 + x.y * a2;
            }
            lr = lr * a1 + l2 * a2;
            mr = M;
          }
        }
        __syncwarp();
        asm volatile("bar.arrive 2, %0;" ::"n"(kNcw * 32));  // slots free again
        const long long te1 = trace ? (long long)globaltimer() : 0;
        const int P0 = pref[s], P1 = pref[s + 1];
        const int c_first = cta_of(P0, T, Gc), c_last = cta_of(P1 - 1, T, Gc);
        const int b = s / p.H, h = s % p.H;
        float* outp = p.out + ((size_t)b * p.Hq + (size_t)h * G) * D;
        if (c_first == c_last) {
          if (g < G) {
            const float inv = lr > 0.f ? 1.f / lr : 0.f;
#pragma unroll
            for (int n = 0; n < D / 8; ++n)
              *reinterpret_cast<float2*>(outp + g * D + n * 8 + 2 * t4) =
                  make_float2(o[n][0] * inv, o[n][1] * inv);
          }
        } else {
          const size_t part = (size_t)blockIdx.x * 2 + ((s == s_first) ? 0 : 1);
          if (g < G) {
#pragma unroll
            for (int n = 0; n < D / 8; ++n)
              *reinterpret_cast<float2*>(p.part_o + (part * 8 + g) * D + n * 8 + 2 * t4) =
                  make_float2(o[n][0], o[n][1]);
            if (t4 == 0) {
              p.part_ml[(part * 2 + 0) * 8 + g] = mr;
              p.part_ml[(part * 2 + 1) * 8 + g] = lr;
            }
          }
          __syncwarp();
          // contributors = CTAs in [c_first, c_last] with a non-empty range; lanes
          // enumerate them 32 at a time
          int n_contrib = 0;
          for (int cb = c_first; cb <= c_last; cb += 32) {
            const int c = cb + lane;
            const bool ok = c <= c_last && cta_start(c, T, Gc) < cta_start(c + 1, T, Gc);
            n_contrib += __popc(__ballot_sync(0xffffffffu, ok));
          }
          int last = 0;
          if (lane == 0) {
            __threadfence();  // release this warp's partial
            last = (atomicAdd(&p.counters[s], 1) == n_contrib - 1);
          }
          last = __shfl_sync(0xffffffffu, last, 0);
          const long long te2 = trace ? (long long)globaltimer() : 0;
          if (trace && lane == 0) trace[9] += te2 - te1;
          if (last) {
            __threadfence();  // acquire the other contributors' partials
            // Merge in CTA order (deterministic). Pass A: row maxima with one
            // contributor per lane. Pass B, for chunks of 4 rows: lanes load the
            // scale factors of their contributor, then every lane streams its
            // D/32 columns of the 4 rows for two contributors per iteration so
            // loads stay in flight instead of serialising on L2 latency.
            constexpr int kCols = D / 32;
            constexpr int kGB = G < 4 ? G : 4;
            using Vec = typename std::conditional<kCols == 4, float4, float2>::type;
            float M[G];
#pragma unroll
            for (int gg = 0; gg < G; ++gg) M[gg] = -INFINITY;
            for (int cb = c_first; cb <= c_last; cb += 32) {
              const int c = cb + lane;
              const int c0s = c <= c_last ? cta_start(c, T, Gc) : 0;
              const bool ok = c <= c_last && c0s < cta_start(c + 1, T, Gc);
              const size_t pc = (size_t)c * 2 + (c0s >= P0 ? 0 : 1);
#pragma unroll
              for (int gg = 0; gg < G; ++gg) {
                float m = ok ? __ldcg(&p.part_ml[(pc * 2 + 0) * 8 + gg]) : -INFINITY;
#pragma unroll
                for (int o2 = 16; o2 > 0; o2 >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o2));
                M[gg] = fmaxf(M[gg], m);
              }
            }
#pragma unroll
            for (int g0 = 0; g0 < G; g0 += kGB) {
              float acc[kGB][kCols];
              float L[kGB];
#pragma unroll
              for (int gg = 0; gg < kGB; ++gg) {
                L[gg] = 0.f;
#pragma unroll
                for (int k = 0; k < kCols; ++k) acc[gg][k] = 0.f;
              }
              for (int cb = c_first; cb <= c_last; cb += 32) {
                const int c = cb + lane;
                const int c0s = c <= c_last ? cta_start(c, T, Gc) : 0;
                const bool ok = c <= c_last && c0s < cta_start(c + 1, T, Gc);
                const int pc = c * 2 + (c0s >= P0 ? 0 : 1);
                float sc[kGB];
#pragma unroll
                for (int gg = 0; gg < kGB; ++gg) {
                  const float Mu = (M[g0 + gg] == -INFINITY) ? 0.f : M[g0 + gg];
                  sc[gg] = ok ? fast_exp2(__ldcg(&p.part_ml[((size_t)pc * 2 + 0) * 8 + g0 + gg]) - Mu) : 0.f;
                  float lw = ok ? __ldcg(&p.part_ml[((size_t)pc * 2 + 1) * 8 + g0 + gg]) * sc[gg] : 0.f;
#pragma unroll
                  for (int o2 = 16; o2 > 0; o2 >>= 1) lw += __shfl_xor_sync(0xffffffffu, lw, o2);
                  L[gg] += lw;
                }
                unsigned mask = __ballot_sync(0xffffffffu, ok);
                while (mask) {  // contributors of this chunk, two at a time, ascending
                  const int a = __ffs(mask) - 1;
                  mask &= mask - 1;
                  const int bl = mask ? __ffs(mask) - 1 : a;
                  const bool has_b = mask != 0;
                  if (has_b) mask &= mask - 1;
                  const int pa = __shfl_sync(0xffffffffu, pc, a);
                  const int pb = __shfl_sync(0xffffffffu, pc, bl);
                  Vec xa[kGB], xb[kGB];
#pragma unroll
                  for (int gg = 0; gg < kGB; ++gg) {
                    xa[gg] = __ldcg(reinterpret_cast<const Vec*>(p.part_o + ((size_t)pa * 8 + g0 + gg) * D) + lane);
                    xb[gg] = __ldcg(reinterpret_cast<const Vec*>(p.part_o + ((size_t)pb * 8 + g0 + gg) * D) + lane);
                  }
#pragma unroll
                  for (int gg = 0; gg < kGB; ++gg) {
                    const float sa = __shfl_sync(0xffffffffu, sc[gg], a);
                    const float sbv = __shfl_sync(0xffffffffu, sc[gg], bl);
                    const float sb = has_b ? sbv : 0.f;
                    acc[gg][0] += xa[gg].x * sa + xb[gg].x * sb;
                    acc[gg][1] += xa[gg].y * sa + xb[gg].y * sb;
                    if constexpr (kCols == 4) {
                      acc[gg][2 % kCols] += xa[gg].z * sa + xb[gg].z * sb;
                      acc[gg][3 % kCols] += xa[gg].w * sa + xb[gg].w * sb;
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
              }
            }
            if (lane == 0) p.counters[s] = 0;
          }
        }
        if (trace && lane == 0) {
          trace[4] += 1;  // emissions
          trace[7] += (long long)globaltimer() - te0;
          trace[8] += te1 - te0;
        }
      }
      fresh = true;
    }
  }
  // consume warp 0's final EMPTY arrival (balances barrier 2 before exit)
  if (warp != 0) asm volatile("bar.sync 2, %0;" ::"n"(kNcw * 32));
  if (trace && threadIdx.x == 0) trace[3] = (long long)globaltimer();
}

using DecodeFn = void (*)(CUtensorMap, CUtensorMap, DecodeParams);

template <int D>
DecodeFn pick_g(int G) {
  switch (G) {
    case 1: return decode_kernel<D, 1>;
    case 2: return decode_kernel<D, 2>;
    case 4: return decode_kernel<D, 4>;
    case 8: return decode_kernel<D, 8>;
    default: return nullptr;
  }
}

}  // namespace

int decode_smem_bytes(int D, int slices) {
  const int fixed = D == 64 ? Geo<64>::kSmemFixed : Geo<128>::kSmemFixed;
  return fixed + (slices + 1) * (int)sizeof(int);
}

int decode_grid(int tiles_upper, int num_sms) { return std::max(1, std::min(2 * num_sms, tiles_upper)); }

cudaError_t launch_decode(const DecodeParams& p, const CUtensorMap& tmk, const CUtensorMap& tmv,
                          int D, int G, int ctas, cudaStream_t stream) {
  DecodeFn fn = (D == 64) ? pick_g<64>(G) : pick_g<128>(G);
  const int S = p.B * p.H;
  if (!fn || S > kMaxSlices || ctas > kMaxCtas) return cudaErrorInvalidValue;
  const int smem = decode_smem_bytes(D, S);
  // raise the dynamic-smem cap once per instantiation to the largest size used
  static int configured[2][9] = {};
  int& cap = configured[D == 64 ? 0 : 1][G];
  if (smem > cap) {
    cudaError_t e = cudaFuncSetAttribute(reinterpret_cast<const void*>(fn),
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    cap = smem;
  }
  return launch_k(fn, dim3(ctas), dim3(kThreads), (size_t)smem, stream, tmk, tmv, p);
}

}  // namespace sfi_impl

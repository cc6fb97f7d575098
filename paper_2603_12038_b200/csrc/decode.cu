// decode.cu — K1 slow-step dense decode (+ pooled-logit emission) and K4
// fast-step sparse decode over the compact cache. One kernel template serves
// both: a (b, kv-head) slice is a list of <= 3 contiguous row segments of a
// bf16 [rows][D] matrix (paged cache for dense; ring + sink/selected rows of
// the compact cache for sparse), split into 64-row tiles, split-KV across
// CTAs, merged with a log-sum-exp combine by the last CTA of each slice.
//
// Reference semantics (paths relative to /root/reference/proj):
//   attend                attention.cpp:80-113   softmax(q.k / sqrt(d)) v
//   dense_segments        attention.cpp:258-268  positions 1..L (current included)
//   sparse_segments       attention.cpp:270-291  compact + recent rows
//   logit capture / pool  attention.cpp:394-409  mean: sum_g logit_g / G; max
//
// B200 design:
//   * a producer warp streams K and V tiles HBM -> smem with TMA
//     (cp.async.bulk.tensor, 128B swizzle) through a STAGES-deep mbarrier ring;
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

#include "common.cuh"
#include "kernels.h"

namespace sfi_impl {

using namespace sfi_dev;

namespace {

constexpr int kTile = 64;   // keys per pipeline stage
constexpr int kNcw = 4;     // consumer warps (16 keys of each tile each)
constexpr int kThreads = (kNcw + 1) * 32;
constexpr int kStages = 3;

template <int D>
struct Geo {
  static constexpr int kBoxes = D / 64;                   // 128-byte TMA boxes per row
  static constexpr int kBoxBytes = kTile * 128;           // 8 KB
  static constexpr int kTileBytes = kBoxes * kBoxBytes;   // one tensor, one tile
  static constexpr int kStageBytes = 2 * kTileBytes;      // K + V
  static constexpr int kSmem = kStages * kStageBytes + 1024 /*align*/ + 256 /*barriers*/;
};

struct Slice {
  int off[3];
  int cnt[3];
  int nseg;
  int tiles;      // total tiles over segments
  int row_base;   // first row of the (layer, b, h) slice in the 2D tensor
  int j_min, j_max;
};

__device__ __forceinline__ int seg_tiles(int c) { return (c + kTile - 1) / kTile; }

// 128B-swizzled address of 16-byte chunk `chunk` (8 bf16) of tile row `row`.
template <int D>
__device__ __forceinline__ uint32_t swz(uint32_t base, int row, int chunk) {
  return base + (chunk >> 3) * Geo<D>::kBoxBytes + row * 128 + (((chunk & 7) ^ (row & 7)) << 4);
}

__device__ __forceinline__ Slice make_slice(const DecodeParams& p, int b, int h) {
  // Segments are fixed slots (0: ring part 1, 1: ring wrap, 2: sink+selected)
  // with count 0 when absent, so every index below is a compile-time constant.
  Slice s;
  const int L = p.prefix_len[b];
  const int nsb = p.n_sink_b[b];
  const int rl = p.recent_len[b];
  s.j_min = nsb + 1;
  s.j_max = L - rl;
  s.off[0] = s.off[1] = s.off[2] = 0;
  s.cnt[0] = s.cnt[1] = s.cnt[2] = 0;
  if (!p.sparse) {
    s.row_base = ((p.layer * p.B + b) * p.H + h) * p.Lmax;
    s.cnt[0] = L > 0 ? L : 0;
  } else {
    s.row_base = ((p.layer * p.B + b) * p.H + h) * p.crows;
    if (rl > 0) {
      const int s0 = (L - rl) % p.R;  // slot of recent_start = L - rl + 1
      const int first = min(rl, p.R - s0);
      s.off[0] = s0;
      s.cnt[0] = first;
      s.cnt[1] = rl - first;
    }
    s.off[2] = p.R;
    s.cnt[2] = nsb + p.n_sel[(p.layer * p.B + b) * p.H + h];
    if (rl > p.R || s.cnt[2] > p.crows - p.R) {  // outside the compact layout
      s.cnt[0] = s.cnt[1] = s.cnt[2] = 0;
      if (h == 0) raise_error(p.err, SFI_ERR_CONFIG);
    }
  }
  s.nseg = 3;
  s.tiles = seg_tiles(s.cnt[0]) + seg_tiles(s.cnt[1]) + seg_tiles(s.cnt[2]);
  return s;
}

// tile index -> (row offset within slice, valid rows)
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

template <int D, int G>
__global__ void __launch_bounds__(kThreads, 2)
    decode_kernel(const __grid_constant__ CUtensorMap tmk, const __grid_constant__ CUtensorMap tmv,
                  const DecodeParams p) {
  static_assert(G >= 1 && G <= 8, "GQA group of at most 8 query heads per KV head");
  static_assert(D == 64 || D == 128, "head_dim 64 or 128");
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * Geo<D>::kStageBytes);
  uint64_t* empty = full + kStages;
  __shared__ int s_last;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int bh = blockIdx.y;
  const int b = bh / p.H, h = bh % p.H;
  const Slice sl = make_slice(p, b, h);
  const int nchunks = min((int)gridDim.x, sl.tiles);
  if ((int)blockIdx.x >= nchunks) {
    if (blockIdx.x == 0 && threadIdx.x == 0) raise_error(p.err, SFI_ERR_EMPTY_SUPPORT);
    return;
  }
  const int per = (sl.tiles + nchunks - 1) / nchunks;
  const int t0 = blockIdx.x * per;
  const int t1 = min(sl.tiles, t0 + per);
  const int ntiles = max(0, t1 - t0);

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kNcw);
    }
    fence_barrier_init();
  }
  __syncthreads();

  if (warp == kNcw) {
    // ---------------- producer: TMA K/V tiles into the stage ring ----------------
    if (lane == 0) {
      tma_prefetch_desc(&tmk);
      tma_prefetch_desc(&tmv);
      const uint64_t pol = l2_policy_evict_first();
      for (int i = 0; i < ntiles; ++i) {
        const int st = i % kStages;
        const uint32_t ph = (i / kStages) & 1;
        mbar_wait(&empty[st], ph ^ 1);
        int off, nv;
        tile_at(sl, t0 + i, off, nv);
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
  } else {
    // ---------------- consumers ----------------
    const int g = lane >> 2, t = lane & 3;
    // Q fragments: rows 0..7 = bf16 hi of query head g (< G), rows 8..15 = lo.
    uint32_t qa[D / 16][4];
    {
      const float* qg = p.q + ((size_t)b * p.Hq + (size_t)h * G + g) * D;
#pragma unroll
      for (int ks = 0; ks < D / 16; ++ks) {
#pragma unroll
        for (int half = 0; half < 2; ++half) {
          const int c = ks * 16 + half * 8 + 2 * t;
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
    }
    float o[D / 8][4];
#pragma unroll
    for (int n = 0; n < D / 8; ++n) o[n][0] = o[n][1] = o[n][2] = o[n][3] = 0.f;
    float m_run = -INFINITY, l_run = 0.f;
    const float sl2 = p.scale_log2;

    for (int i = 0; i < ntiles; ++i) {
      const int st = i % kStages;
      const uint32_t ph = (i / kStages) & 1;
      int off, nv;
      tile_at(sl, t0 + i, off, nv);
      mbar_wait(&full[st], ph);
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
        float s[2][2];
        bool valid[2][2];
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            s[j][e] = acc[j][e] + acc[j][e + 2];
            valid[j][e] = (kw + j * 8 + 2 * t + e) < nv;
          }
        // ---- pooled logits over J (dense slow step) ----
        if (p.logits != nullptr) {
          const int pos0 = off + kw + 1;  // dense row r holds position r + 1
          if (pos0 + 15 >= sl.j_min && pos0 <= sl.j_max) {
#pragma unroll
            for (int j = 0; j < 2; ++j)
#pragma unroll
              for (int e = 0; e < 2; ++e) {
                float v = s[j][e] * p.inv_sqrt_d;
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
                const int pos = pos0 + j * 8 + 2 * t + e;
                if (g == 0 && valid[j][e] && pos >= sl.j_min && pos <= sl.j_max)
                  p.logits[(size_t)bh * p.Lmax + (pos - sl.j_min)] = v;
              }
          }
        }
        // ---- online softmax (log2 domain) ----
        float mx = -INFINITY;
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            s[j][e] = valid[j][e] ? s[j][e] * sl2 : -INFINITY;
            mx = fmaxf(mx, s[j][e]);
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
            pr[j][e] = fast_exp2(s[j][e] - m_use);
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
    }

    // ---- warp partial -> smem (reuses the stage ring; all TMA traffic has landed) ----
    l_run += __shfl_xor_sync(0xffffffffu, l_run, 1);
    l_run += __shfl_xor_sync(0xffffffffu, l_run, 2);
    float* red_o = reinterpret_cast<float*>(smem);                  // [kNcw][G][D]
    float* red_ml = red_o + kNcw * G * D;                           // [kNcw][2][G]
    // make sure every consumer warp finished reading the ring before reuse
    asm volatile("bar.sync 1, %0;" ::"n"(kNcw * 32));
    if (g < G) {
#pragma unroll
      for (int n = 0; n < D / 8; ++n) {
        const int c = n * 8 + 2 * t;
        red_o[(warp * G + g) * D + c] = o[n][0] + o[n][2];
        red_o[(warp * G + g) * D + c + 1] = o[n][1] + o[n][3];
      }
      if (t == 0) {
        red_ml[(warp * 2 + 0) * G + g] = m_run;
        red_ml[(warp * 2 + 1) * G + g] = l_run;
      }
    }
  }
  __syncthreads();

  // ---- combine warps; write the chunk partial or the final output ----
  const float* red_o = reinterpret_cast<const float*>(smem);
  const float* red_ml = red_o + kNcw * G * D;
  float* outp = p.out + ((size_t)b * p.Hq + (size_t)h * G) * D;
  const bool single = (nchunks == 1);
  const size_t part = (size_t)bh * p.max_chunks + blockIdx.x;
  for (int idx = threadIdx.x; idx < G * D; idx += kThreads) {
    const int gg = idx / D;
    float M = -INFINITY;
#pragma unroll
    for (int w = 0; w < kNcw; ++w) M = fmaxf(M, red_ml[(w * 2) * G + gg]);
    const float Mu = (M == -INFINITY) ? 0.f : M;
    float acc = 0.f, L = 0.f;
#pragma unroll
    for (int w = 0; w < kNcw; ++w) {
      const float sc = fast_exp2(red_ml[(w * 2) * G + gg] - Mu);
      acc += red_o[(w * G + gg) * D + (idx % D)] * sc;
      L += red_ml[(w * 2 + 1) * G + gg] * sc;
    }
    if (single) {
      outp[idx] = L > 0.f ? acc / L : 0.f;
    } else {
      p.part_o[part * G * D + idx] = acc;
      if (idx % D == 0) {
        p.part_ml[(part * 2 + 0) * 8 + gg] = M;
        p.part_ml[(part * 2 + 1) * 8 + gg] = L;
      }
    }
  }
  if (single) return;

  // ---- split-KV merge by the last-arriving CTA of this slice ----
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = (atomicAdd(&p.counters[bh], 1) == nchunks - 1);
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  const size_t part0 = (size_t)bh * p.max_chunks;
  for (int idx = threadIdx.x; idx < G * D; idx += kThreads) {
    const int gg = idx / D;
    float M = -INFINITY;
    for (int c = 0; c < nchunks; ++c) M = fmaxf(M, __ldcg(&p.part_ml[((part0 + c) * 2) * 8 + gg]));
    const float Mu = (M == -INFINITY) ? 0.f : M;
    float acc = 0.f, L = 0.f;
    for (int c = 0; c < nchunks; ++c) {
      const float sc = fast_exp2(__ldcg(&p.part_ml[((part0 + c) * 2) * 8 + gg]) - Mu);
      acc += __ldcg(&p.part_o[(part0 + c) * G * D + idx]) * sc;
      L += __ldcg(&p.part_ml[((part0 + c) * 2 + 1) * 8 + gg]) * sc;
    }
    outp[idx] = L > 0.f ? acc / L : 0.f;
    if (L <= 0.f && idx == 0) raise_error(p.err, SFI_ERR_EMPTY_SUPPORT);
  }
  if (threadIdx.x == 0) p.counters[bh] = 0;
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

int decode_smem_bytes(int D) { return D == 64 ? Geo<64>::kSmem : Geo<128>::kSmem; }

// Chunks per (b, head) slice: fill the machine with 2 CTAs/SM in as close
// to a whole number of waves as possible, at least 2 tiles per CTA.
int choose_chunks(int slices, int tiles_per_slice, int num_sms) {
  const int slots = 2 * num_sms;
  int best = 1;
  double best_score = -1.0;
  const int cmax = std::max(1, std::min(kMaxChunks, tiles_per_slice / 2));
  for (int c = 1; c <= cmax; ++c) {
    const double waves = double(slices) * c / slots;
    const double eff = waves / std::ceil(waves);
    if (waves > 4.0 && c > 1) break;
    const double score = eff - 0.004 * c;
    if (score > best_score + 1e-9) {
      best_score = score;
      best = c;
    }
  }
  return best;
}

cudaError_t launch_decode(const DecodeParams& p, const CUtensorMap& tmk, const CUtensorMap& tmv,
                          int D, int G, int chunks, cudaStream_t stream) {
  DecodeFn fn = (D == 64) ? pick_g<64>(G) : pick_g<128>(G);
  if (!fn) return cudaErrorInvalidValue;
  const int smem = decode_smem_bytes(D);
  cudaError_t e = cudaFuncSetAttribute(reinterpret_cast<const void*>(fn),
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  dim3 grid(chunks, p.B * p.H);
  fn<<<grid, kThreads, smem, stream>>>(tmk, tmv, p);
  return cudaGetLastError();
}

}  // namespace sfi_impl

// fast_decode.cu — K4: the fast-step sparse decode over the compact cache,
// optionally fused with the current token's append (K3a) so a fast step is
// ONE launch per layer.
//
// Reference semantics (paths relative to /root/reference/proj):
//   sparse_segments       attention.cpp:270-291  compact rows (sink + selected)
//                                                then the recent tail
//   attend                attention.cpp:80-113   softmax(q.k / sqrt(d)) v
//   KvStore::append_layer attention.cpp:136-152  row L-1 <- k, v; fp64 key norm
//                                                summed in c order
//   run_step              attention.cpp:354-360  the token is appended before
//                                                attention, so it attends to itself
//
// B200 design:
//   * one thread-block cluster of C CTAs per (b, kv head) slice; the slice's
//     compact rows [0, R) (recent ring) and [R, R + n_sink_b + n_sel) (sink +
//     selected) are cut into 64-row tiles and split evenly over the C CTAs;
//   * SFI_FAST_STEAL=1 (opt-in): the producers claim tiles from a per-slice
//     counter in L2 instead (intra-cluster balancing of HBM service variance;
//     -2.4% per C2 layer, slower where a CTA has only 1-3 tiles). The
//     summation order then varies run to run, so the static split stays the
//     default (deterministic outputs);
//   * the tile split depends only on n_sink_b / n_sel, which no kernel of a fast
//     step writes, so with SFI_FAST_PREFETCH the TMA producer issues its first
//     stages BEFORE the programmatic-dependent-launch wait: the K/V stream of
//     layer l starts while layer l-1's kernel drains;
//   * producer warp: TMA (128B swizzle, L2 evict-first) into a 3-stage mbarrier
//     ring; 4 consumer warps: QK^T and PV with mma.sync m16n8k16 bf16 -> fp32
//     (query rows = the G heads of the GQA group, bf16 hi/lo split so the fp32
//     query keeps ~16 mantissa bits), online softmax in the log2 domain with
//     lazy rescaling of the running max;
//   * aux warp (cluster rank 0): the current token. Its K/V come from the
//     caller's k_new / v_new: it persists them (paged row L-1, ring slot
//     (L-1) % R, fp64 norm — bit-identical to sfi_ring_append) and contributes
//     the token's key as one more softmax partial; the ring slot's stale row is
//     masked out of the tiles, so no CTA ever reads a row this kernel writes;
//   * merge: each CTA combines its 5 partials (m, l, O) locally, then PUSHES
//     the combined partial to the owners with st.async remote stores that
//     complete_tx on the owner's receive mbarrier (owner r merges a warp-aligned
//     1/C share of the G x D outputs; with G <= 4 and C <= 4 rank 0 merges all
//     and the others exit right after pushing). No cluster barrier on the merge
//     path: the owner waits on its own mbarrier, then merges from its shared
//     memory in one pass (fixed order: deterministic). A phase-0 cluster
//     arrive / wait at start guarantees every peer runs before it is written;
//     no exit barrier: once pushed, no CTA touches a peer.
#include <cooperative_groups.h>
#include <cuda.h>

#include <algorithm>
#include <cmath>

#include "common.cuh"
#include "kernels.h"

namespace cg = cooperative_groups;

namespace sfi_impl {

using namespace sfi_dev;

namespace {

constexpr int kTile = 64;
constexpr int kNcw = 4;                        // consumer warps
constexpr int kThreads = (kNcw + 2) * 32;      // + producer warp + aux warp
constexpr int kStages = 3;
constexpr int kParts = kNcw + 1;               // softmax partials per CTA

template <int D>
struct FGeo {
  static constexpr int kBoxes = D / 64;
  static constexpr int kBoxBytes = kTile * 128;
  static constexpr int kTileBytes = kBoxes * kBoxBytes;
  static constexpr int kStageBytes = 2 * kTileBytes;
  static constexpr int kRing = kStages * kStageBytes;
};

template <int D, int G>
struct FPart {  // partials, written over the (drained) stage ring
  static constexpr int kPD = D + 8;               // row stride: the mma-layout stores hit 8 rows at once
  static constexpr int kO = kParts * G * kPD;     // floats
  static constexpr int kBytes = (kO + 3 * kParts * G + 2 * G) * 4;
  static_assert(kBytes <= FGeo<D>::kRing, "partials must fit in the stage ring");
};
// Merge receive area (dedicated: CTAs push into it while the owner may still be
// streaming): [C][share] combined O + [C][G] m + [C][G] l, share <= G*D/C + 32.
template <int D, int G>
struct FRecv {
  // O area: C x share floats; a single owner (G <= 4, C <= 4) takes all C partials;
  // then m, l [16][G]
  static constexpr int kO = (G <= 4 && 4 * G * D > G * D + 32 * 16) ? 4 * G * D : G * D + 32 * 16;
  static constexpr int kFloats = kO + 2 * 16 * G;
};
template <int D, int G>
__host__ __device__ constexpr int fast_smem_off_tiles() {  // [kStages] tile index of each stage (dynamic split)
  return FGeo<D>::kRing + 64 + D * 8 + FRecv<D, G>::kFloats * 4;
}
template <int D, int G>
constexpr int fast_smem_bytes() {  // stage ring | 2 x kStages mbarriers | fp64 k^2 row | receive area | stage tiles
  return fast_smem_off_tiles<D, G>() + 16;
}
// Owner shares are whole warps of 32 elements. With few, small partials (G <= 4,
// C <= 4) rank 0 merges everything and ranks 1.. exit right after their push,
// freeing their SM slots for the next layer's CTAs (its prefetch starts early).
__host__ __device__ constexpr int merge_share(int G, int D, int C) {
  return (G <= 4 && C <= 4) ? ((G * D + 31) & ~31) : ((G * D + C - 1) / C + 31) & ~31;
}
// Bytes owner r receives: from each of the C CTAs its O over [e0, e1) and
// (m, l) of every head that range touches.
__host__ __device__ constexpr uint32_t merge_rx_bytes(int G, int D, int C, int r) {
  const int share = merge_share(G, D, C);
  const int e0 = r * share, e1 = (e0 + share < G * D) ? e0 + share : G * D;
  return e1 > e0 ? (uint32_t)C * (uint32_t)((e1 - e0) * 4 + ((e1 - 1) / D - e0 / D + 1) * 8) : 0u;
}

template <int D>
__device__ __forceinline__ uint32_t swz(uint32_t base, int row, int chunk) {
  return base + (chunk >> 3) * FGeo<D>::kBoxBytes + row * 128 + (((chunk & 7) ^ (row & 7)) << 4);
}

// Phase 0 of the cluster barrier: every CTA arrives when it starts and waits
// just before its first remote store, so no CTA writes into a peer that has not
// started.
__device__ __forceinline__ void cluster_arrive_started() {
  __syncwarp();
  asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait_started() {
  __syncwarp();
  asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
}

// Tile t of a slice (ring tiles first) -> first compact row.
__device__ __forceinline__ int tile_row(int t, int t_ring, int R) {
  return t < t_ring ? t * kTile : R + (t - t_ring) * kTile;
}

// CTA-local combine of the kParts warp partials (160 threads: consumers + aux):
// first the per-head (M, scales, L) — G threads, written to comb_m / comb_l /
// part_s — then O into part 0 in place, four elements per thread per pass.
template <int D, int G>
__device__ __forceinline__ void combine_cta(float* part_o, const float* part_m, const float* part_l,
                                            float* comb_m, float* comb_l, float* part_s, int tid) {
  constexpr int kT = (kNcw + 1) * 32;
  constexpr int kPD = FPart<D, G>::kPD;
  if (tid < G) {
    float m[kParts], M = -INFINITY;
#pragma unroll
    for (int w = 0; w < kParts; ++w) {
      m[w] = part_m[w * G + tid];
      M = fmaxf(M, m[w]);
    }
    const float Mu = (M == -INFINITY) ? 0.f : M;
    float Ls = 0.f;
#pragma unroll
    for (int w = 0; w < kParts; ++w) {
      const float l = part_l[w * G + tid];
      const float sc = l > 0.f ? fast_exp2(m[w] - Mu) : 0.f;  // l == 0: partial O is zero
      part_s[w * G + tid] = sc;
      Ls += l * sc;
    }
    comb_m[tid] = M;
    comb_l[tid] = Ls;
  }
  named_bar_sync<3, kT>();
#pragma unroll 2
  for (int e = tid * 4; e < G * D; e += kT * 4) {
    const int g = e / D;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int w = 0; w < kParts; ++w) {
      const float sc = part_s[w * G + g];
      const float4 x = *reinterpret_cast<const float4*>(part_o + (w * G + g) * kPD + (e - g * D));
      acc.x = fmaf(x.x, sc, acc.x);
      acc.y = fmaf(x.y, sc, acc.y);
      acc.z = fmaf(x.z, sc, acc.z);
      acc.w = fmaf(x.w, sc, acc.w);
    }
    *reinterpret_cast<float4*>(part_o + g * kPD + (e - g * D)) = acc;
  }
}

// Push this CTA's combined partial to the owners (160 threads, after
// combine_cta): owner r merges elements [r*share, (r+1)*share) and receives, in
// slot `rank`, this CTA's O for them (float4 remote stores) and (m, l) of their
// heads.
template <int D, int G>
__device__ __forceinline__ void push_partials(const float* part_o, const float* comb_m, const float* comb_l,
                                              float* recv_o, float* recv_m, float* recv_l, uint64_t* rx_bar,
                                              int share, int rank, int tid) {
  constexpr int kT = (kNcw + 1) * 32;
  constexpr int kPD = FPart<D, G>::kPD;
  named_bar_sync<3, kT>();  // combined O complete (phase 0 was waited for before griddep_wait)
  const uint32_t bar = smem_u32(rx_bar);
  for (int e = tid * 4; e < G * D; e += kT * 4) {
    const int r = e / share;  // share is a multiple of 32: a float4 never straddles owners
    const int g = e / D;
    const float4 v = *reinterpret_cast<const float4*>(part_o + g * kPD + (e - g * D));
    st_async_v4(mapa_shared(smem_u32(recv_o + rank * share + (e - r * share)), r), v, mapa_shared(bar, r));
  }
  if (tid < G) {
    const int r0 = (tid * D) / share, r1 = ((tid + 1) * D - 1) / share;
    for (int r = r0; r <= r1; ++r) {
      const uint32_t rb = mapa_shared(bar, r);
      st_async_f32(mapa_shared(smem_u32(recv_m + rank * G + tid), r), comb_m[tid], rb);
      st_async_f32(mapa_shared(smem_u32(recv_l + rank * G + tid), r), comb_l[tid], rb);
    }
  }
}

// The owner's merge, once its receive mbarrier has seen every pushed byte.
// Everything is re-derived from special registers, kernel parameters and
// shared memory (no long-lived registers across the wait).
template <int D, int G>
__device__ __forceinline__ void merge_pushed(const FastParams& p, uint8_t* smem) {
  const int C = (int)sreg_cluster_nctarank();
  const int rank = (int)sreg_cluster_ctarank();
  const int tid = (int)sreg_tid_x();
  const int s = (int)sreg_ctaid_x() / C;
  const int b = s / p.H, h = s % p.H;
  const int share = merge_share(G, D, C);
  const float* recv_o = reinterpret_cast<const float*>(smem + FGeo<D>::kRing + 64 + D * 8);
  const float* recv_m = recv_o + FRecv<D, G>::kO;
  const float* recv_l = recv_m + 16 * G;
  const bool ok = *reinterpret_cast<const int*>(smem + FGeo<D>::kRing + 48) != 0;
  long long* trace = p.trace ? p.trace + (size_t)sreg_ctaid_x() * 16 : nullptr;
  const long long c_pub0 = clock64();
  mbar_wait(reinterpret_cast<uint64_t*>(smem + FGeo<D>::kRing + 56), 0);  // every partial landed
  if (trace && tid == 0) {
    trace[4] = clock64() - c_pub0;  // receive-wait cycles
    trace[13] = (long long)globaltimer();
  }
  const long long c_merge0 = clock64();

  // ---- merge: this CTA's share [e0, e1) of the G x D outputs over the C pushed partials ----
  // One pass, no barrier: each thread owns float4s of outputs and forms its
  // head's max, scales and L itself from the C (m, l) pairs (fixed c order:
  // deterministic), accumulating sum_c O_c * scale_c alongside.
  const int total = G * D;
  const int e0 = rank * share, e1 = min(total, e0 + share);
  float* outp = p.out + ((size_t)b * p.Hq + (size_t)h * G) * D;
  for (int e = e0 + tid * 4; e < e1; e += kNcw * 32 * 4) {
    const int g = e / D;
    float M = -INFINITY;
#pragma unroll 4
    for (int c = 0; c < C; ++c) M = fmaxf(M, recv_m[c * G + g]);
    const float Mu = (M == -INFINITY) ? 0.f : M;
    float L = 0.f;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 4
    for (int c = 0; c < C; ++c) {
      const float l = recv_l[c * G + g];
      const float sc = l > 0.f ? fast_exp2(recv_m[c * G + g] - Mu) : 0.f;  // l == 0: that CTA's O is zero
      L += l * sc;
      const float4 x = *reinterpret_cast<const float4*>(recv_o + c * share + (e - e0));
      acc.x = fmaf(x.x, sc, acc.x);
      acc.y = fmaf(x.y, sc, acc.y);
      acc.z = fmaf(x.z, sc, acc.z);
      acc.w = fmaf(x.w, sc, acc.w);
    }
    const float inv = L > 0.f ? 1.f / L : 0.f;
    *reinterpret_cast<float4*>(outp + e) = make_float4(acc.x * inv, acc.y * inv, acc.z * inv, acc.w * inv);
    if (e % D == 0) {
      if (p.lse) {  // partial mode (sequence shard): natural-log LSE, empty allowed
        p.lse[(size_t)b * p.Hq + (size_t)h * G + g] = L > 0.f ? (M + __log2f(L)) * 0.69314718055994531f : -INFINITY;
      } else if (rank == 0 && e == 0 && ok && !(L > 0.f)) {
        raise_error(p.err, SFI_ERR_EMPTY_SUPPORT);
      }
    }
  }
  if (trace && tid == 0) {
    trace[7] = clock64() - c_merge0;  // merge cycles
    trace[14] = (long long)globaltimer();
    trace[3] = (long long)globaltimer();
  }
}

template <int D, int G>
__global__ void __launch_bounds__(kThreads, 2)
    fast_decode_kernel(const __grid_constant__ CUtensorMap tmk, const __grid_constant__ CUtensorMap tmv,
                       const FastParams p) {
  static_assert(G == 1 || G == 2 || G == 4 || G == 8 || G == 16, "GQA group 1..16");
  static_assert(D == 64 || D == 128, "head_dim 64 or 128");
  constexpr int NH = (G == 16) ? 2 : 1;   // query heads per mma row-thread
  constexpr int NQ = (G == 16) ? 2 : 1;   // A-operand blocks (hi / lo) per k-step
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + FGeo<D>::kRing);
  uint64_t* empty = full + kStages;
  uint64_t* rx_bar = reinterpret_cast<uint64_t*>(smem + FGeo<D>::kRing + 56);  // merge receive (flag at +48)
  volatile int* stage_tile = reinterpret_cast<volatile int*>(smem + fast_smem_off_tiles<D, G>());
  constexpr int kPD = FPart<D, G>::kPD;
  float* part_o = reinterpret_cast<float*>(smem);        // [kParts][G][kPD] (after the stream)
  float* part_m = part_o + FPart<D, G>::kO;              // [kParts][G]
  float* part_l = part_m + kParts * G;                   // [kParts][G]
  float* comb_m = part_l + kParts * G;                   // [G] CTA-combined (m, l);
  float* comb_l = comb_m + G;                            //     O combined in place in part 0
  float* part_s = comb_l + G;                            // [kParts][G] combine scales
  double* ksq = reinterpret_cast<double*>(smem + FGeo<D>::kRing + 64);  // [D] k_c^2 (aux)
  float* recv_o = reinterpret_cast<float*>(smem + FGeo<D>::kRing + 64 + D * 8);  // [C][share]
  float* recv_m = recv_o + FRecv<D, G>::kO;                                      // [C][G]
  float* recv_l = recv_m + 16 * G;                                               // [C][G]

  long long* trace = p.trace ? p.trace + (size_t)blockIdx.x * 16 : nullptr;
  if (trace && threadIdx.x == 0) {
    trace[0] = (long long)globaltimer();
    trace[6] = smid();
  }
  cg::cluster_group cl = cg::this_cluster();
  const int C = (int)cl.num_blocks();
  const int rank = (int)cl.block_rank();
  const int s = blockIdx.x / C;          // slice = b * H + h
  const int b = s / p.H, h = s % p.H;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const size_t slice_g = (size_t)(p.layer * p.B + b) * p.H + h;  // (layer, b, h)

  if (threadIdx.x == kNcw * 32) {
    tma_prefetch_desc(&tmk);
    tma_prefetch_desc(&tmv);
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i < kStages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], kNcw);
    }
    mbar_init(rx_bar, 1);
    fence_barrier_init();
    // the owner's one arrival: the bytes the C peers will push (complete_tx may
    // land before or after it; the phase completes when both balance)
    mbar_arrive_expect_tx(rx_bar, merge_rx_bytes(G, D, C, rank));
  }
  // Static tile split over the compact layout [0, R) + [R, R + n_sink + K):
  // no global load before the producer's first TMA. In steady-state decode
  // n_sel = K, so it equals the live split; shorter selections only leave
  // masked rows in the last tiles.
  const int t_ring = (p.R + kTile - 1) / kTile;
  const int T = t_ring + (p.crows - p.R + kTile - 1) / kTile;
  const int tb = (int)(((long long)rank * T) / C), te = (int)(((long long)(rank + 1) * T) / C);
  const int row_base = (int)(slice_g * p.crows);
  const int share = merge_share(G, D, C);
  __syncthreads();
  cluster_arrive_started();  // phase 0: this CTA runs (its receive area may be written)

  if (warp == kNcw) {
    // ---------------- producer ----------------
    if (lane == 0) {
      if (!p.prefetch) griddep_wait();  // the compact rows may come from the predecessor
      const uint64_t pol = l2_policy_evict_first();
      // dynamic split (p.steal): tiles are claimed from the slice's counter in
      // L2; a claim past T ends the stream with an empty stage (tile -1)
      int32_t* claim = p.steal ? p.steal + slice_g * 2 : nullptr;
      for (int t = tb, i = 0;; ++t, ++i) {
        if (claim) {
          if (i == kStages) griddep_wait();
        } else if (t >= te) {
          break;
        } else if (i == kStages) {
          griddep_wait();  // the rest needs freed stages anyway
        }
        const int st = i % kStages;
        const uint32_t ph = (i / kStages) & 1;
        mbar_wait(&empty[st], ph ^ 1);
        if (claim) {
          t = atomicAdd(claim, 1);
          stage_tile[st] = t < T ? t : -1;
          if (t >= T) {  // end of stream: release the consumers without data
            mbar_arrive(&full[st]);
            if (atomicAdd(claim + 1, 1) == C - 1) {  // last producer of the cluster: reset
              claim[0] = 0;
              claim[1] = 0;
            }
            break;
          }
        }
        const int row = row_base + tile_row(t, t_ring, p.R);
        uint8_t* kdst = smem + st * FGeo<D>::kStageBytes;
        uint8_t* vdst = kdst + FGeo<D>::kTileBytes;
        mbar_arrive_expect_tx(&full[st], FGeo<D>::kStageBytes);
#pragma unroll
        for (int bx = 0; bx < FGeo<D>::kBoxes; ++bx) {
          tma_load_2d(kdst + bx * FGeo<D>::kBoxBytes, &tmk, bx * 64, row, &full[st], pol);
          tma_load_2d(vdst + bx * FGeo<D>::kBoxBytes, &tmv, bx * 64, row, &full[st], pol);
        }
      }
    }
    __syncwarp();
    if (trace && lane == 0) trace[10] = (long long)globaltimer();
    griddep_wait();
    griddep_launch();
    cluster_wait_started();
    return;
  }

  cluster_wait_started();  // off the critical path: under PDL this CTA waits for its predecessor anyway
  griddep_wait();
  griddep_launch();
  if (trace && threadIdx.x == 0) {
    trace[1] = (long long)globaltimer();
    trace[5] = te - tb;
  }
  // post-wait: lengths of this step (loads issued here; the consumers derive
  // from them only after issuing their q loads, so both round trips overlap)
  const int L = p.prefix_len[b];
  const int rl = p.recent_len[b];
  const int nsb = p.n_sink_b[b];
  const int nsel = p.n_sel[slice_g];
  const bool fused = p.k_new != nullptr;
#define SFI_FAST_DERIVE_LENGTHS                                                                    \
  const int n_cs = nsb + nsel; /* sink + selected rows */                                          \
  const bool geom_ok = nsb >= 0 && nsel >= 0 && n_cs <= p.crows - p.R;                             \
  /* ring slots holding the recent window minus (fused) the current token */                       \
  const int s0 = ((L - rl) % p.R + p.R) % p.R; /* slot of recent_start = L - rl + 1 */             \
  const int ring_valid = fused ? rl - 1 : rl;                                                      \
  const bool ok = geom_ok && rl <= p.R && rl >= (fused ? 1 : 0) && L >= 1 && L <= p.Lmax;

  if (warp == kNcw + 1) {
    SFI_FAST_DERIVE_LENGTHS
    // ---------------- aux: the current token ----------------
    constexpr int kC = D / 32;
    float mq[G], lq[G];
    float vv[kC];
#pragma unroll
    for (int g = 0; g < G; ++g) {
      mq[g] = -INFINITY;
      lq[g] = 0.f;
    }
#pragma unroll
    for (int c = 0; c < kC; ++c) vv[c] = 0.f;
    const bool mine = rank == 0 && ok && fused && !overflow_raised(p.err);
    if (rank == 0 && !ok && lane == 0)
      raise_error(p.err, (rl < 1 && fused) || L < 1 || L > p.Lmax ? SFI_ERR_OUT_OF_RANGE : SFI_ERR_CONFIG);
    if (mine) {
      const size_t src = ((size_t)b * p.H + h) * D + lane * kC;
      __nv_bfloat16 kx[kC], vx[kC];
      float qv[G][kC];
#pragma unroll
      for (int c = 0; c < kC; ++c) {
        kx[c] = p.k_new[src + c];
        vx[c] = p.v_new[src + c];
      }
#pragma unroll
      for (int g = 0; g < G; ++g)
#pragma unroll
        for (int c = 0; c < kC; ++c) qv[g][c] = p.q[((size_t)b * p.Hq + (size_t)h * G + g) * D + lane * kC + c];
      // persist: paged row L-1, ring slot (L-1) % R (attention.cpp:141-142)
      const size_t prow = (slice_g * p.Lmax + (L - 1)) * D + lane * kC;
      const size_t rrow = (slice_g * p.crows + (L - 1) % p.R) * D + lane * kC;
#pragma unroll
      for (int c = 0; c < kC; ++c) {
        p.kc[prow + c] = kx[c];
        p.vc[prow + c] = vx[c];
        p.ck[rrow + c] = kx[c];
        p.cv[rrow + c] = vx[c];
        const double x = (double)__bfloat162float(kx[c]);
        ksq[lane * kC + c] = __dmul_rn(x, x);  // exact: bf16^2 fits in fp64
        vv[c] = __bfloat162float(vx[c]);
      }
      // the token's key as one more partial: m = q.k * log2(e)/sqrt(d), l = 1, O = v
#pragma unroll
      for (int g = 0; g < G; ++g) {
        float d0 = 0.f;
#pragma unroll
        for (int c = 0; c < kC; ++c) d0 += qv[g][c] * __bfloat162float(kx[c]);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) d0 += __shfl_xor_sync(0xffffffffu, d0, o);
        mq[g] = d0 * p.scale_log2;
        lq[g] = 1.f;
      }
    }
    if (trace && lane == 0) trace[8] = (long long)globaltimer();
    named_bar_sync<1, (kNcw + 1) * 32>();  // stage ring drained
#pragma unroll
    for (int g = 0; g < G; ++g) {
#pragma unroll
      for (int c = 0; c < kC; ++c) part_o[(kNcw * G + g) * kPD + lane * kC + c] = (lq[g] > 0.f) ? vv[c] : 0.f;
      if (lane == 0) {
        part_m[kNcw * G + g] = mq[g];
        part_l[kNcw * G + g] = lq[g];
      }
    }
    named_bar_sync<2, (kNcw + 1) * 32>();  // all partials written
    combine_cta<D, G>(part_o, part_m, part_l, comb_m, comb_l, part_s, (int)threadIdx.x - 32);
    push_partials<D, G>(part_o, comb_m, comb_l, recv_o, recv_m, recv_l, rx_bar, share, rank, (int)threadIdx.x - 32);
    // fp64 key norm: sequential over c in round-to-nearest ops (attention.cpp:
    // 143-150; bit-identical to append_kernel), off the critical path
    if (mine && lane == 0) {
      double acc = 0.0;
#pragma unroll 16
      for (int c = 0; c < D; ++c) acc = __dadd_rn(acc, ksq[c]);
      p.norms[slice_g * p.Lmax + (L - 1)] = __dsqrt_rn(acc);
    }
    return;
  }

  // ---------------- consumers ----------------
  const int g = lane >> 2, t4 = lane & 3;
  // Q fragments. G <= 8: rows 0..7 = bf16 hi of head g, rows 8..15 = lo.
  // G == 16: block 0 = hi of heads 0..15, block 1 = lo.
  uint32_t qa[NQ][D / 16][4];
  {
    const float* qb = p.q + ((size_t)b * p.Hq + (size_t)h * G) * D;
#pragma unroll
    for (int ks = 0; ks < D / 16; ++ks)
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        const int c = ks * 16 + half * 8 + 2 * t4;
        if constexpr (G == 16) {
#pragma unroll
          for (int r = 0; r < 2; ++r) {  // r: row g (head g) / row g + 8 (head g + 8)
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
  SFI_FAST_DERIVE_LENGTHS
#undef SFI_FAST_DERIVE_LENGTHS
  float o[D / 8][4];
#pragma unroll
  for (int n = 0; n < D / 8; ++n) o[n][0] = o[n][1] = o[n][2] = o[n][3] = 0.f;
  float m_run[NH], l_run[NH];
#pragma unroll
  for (int i = 0; i < NH; ++i) {
    m_run[i] = -INFINITY;
    l_run[i] = 0.f;
  }
  const float sl2 = p.scale_log2;
  const int kw = warp * 16;

  // every tile is waited for and released even when the step is invalid, so
  // the producer never blocks and no TMA write is in flight at exit
  for (int t = tb, i = 0;; ++t, ++i) {
    const int st = i % kStages;
    const uint32_t ph = (i / kStages) & 1;
    if (p.steal) {  // the producer's claim for this stage, published before its full arrival
      mbar_wait(&full[st], ph);
      t = stage_tile[st];
      if (t < 0) break;
    } else if (t >= te) {
      break;
    }
    // validity of this warp's keys kw + j*8 + 2*t4 + e
    bool valid[2][2];
    const bool ring = t < t_ring;
    const int r0 = tile_row(t, t_ring, p.R) + kw;
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int r = r0 + j * 8 + 2 * t4 + e;
        if (ring) {
          int dlt = r - s0;
          if (dlt < 0) dlt += p.R;
          valid[j][e] = r < p.R && dlt < ring_valid;
        } else {
          valid[j][e] = (r - p.R) < n_cs;
        }
      }
    const bool any =
        __any_sync(0xffffffffu, ok && (valid[0][0] | valid[0][1] | valid[1][0] | valid[1][1]));
    if (!p.steal) mbar_wait(&full[st], ph);
    if (trace && i == 0 && threadIdx.x == 0) trace[2] = (long long)globaltimer();
    if (any) {
      const uint32_t kbase = smem_u32(smem + st * FGeo<D>::kStageBytes);
      const uint32_t vbase = kbase + FGeo<D>::kTileBytes;
      float acc[2][4];
#pragma unroll
      for (int j = 0; j < 2; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.f;
#pragma unroll
      for (int kc = 0; kc < D / 16; kc += 2) {
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          uint32_t b0, b1, b2, b3;
          ldsm_x4(swz<D>(kbase, kw + j * 8 + (lane & 7), kc * 2 + (lane >> 3)), b0, b1, b2, b3);
#pragma unroll
          for (int qb = 0; qb < NQ; ++qb) {
            mma_bf16(acc[j], qa[qb][kc], b0, b1);
            mma_bf16(acc[j], qa[qb][kc + 1], b2, b3);
          }
        }
      }
      // scores of head(s) of this thread, log2 domain
      float sc[NH][2][2];
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
#pragma unroll
          for (int hh = 0; hh < NH; ++hh) sc[hh][j][e] = valid[j][e] ? sc[hh][j][e] * sl2 : -INFINITY;
        }
      float pr[NH][2][2], alpha[NH];
      bool any_grow = false;
#pragma unroll
      for (int hh = 0; hh < NH; ++hh) {
        float mx = fmaxf(fmaxf(sc[hh][0][0], sc[hh][0][1]), fmaxf(sc[hh][1][0], sc[hh][1][1]));
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
      // P as the A operand (see header): G <= 8 rows g / g+8 = hi / lo of head g;
      // G == 16 block 0 = hi of heads (g, g+8), block 1 = lo.
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
  }

  // ---- publish this warp's partial over the drained stage ring ----
#pragma unroll
  for (int hh = 0; hh < NH; ++hh) {
    l_run[hh] += __shfl_xor_sync(0xffffffffu, l_run[hh], 1);
    l_run[hh] += __shfl_xor_sync(0xffffffffu, l_run[hh], 2);
  }
  if (trace && threadIdx.x == 0) trace[9] = (long long)globaltimer();
  named_bar_sync<1, (kNcw + 1) * 32>();
  if (trace && threadIdx.x == 0) trace[12] = (long long)globaltimer();
  if constexpr (NH == 2) {
#pragma unroll
    for (int hh = 0; hh < 2; ++hh) {
      float* dst = part_o + (warp * G + g + 8 * hh) * kPD;
#pragma unroll
      for (int n = 0; n < D / 8; ++n)
        *reinterpret_cast<float2*>(dst + n * 8 + 2 * t4) = make_float2(o[n][2 * hh], o[n][2 * hh + 1]);
      if (t4 == 0) {
        part_m[warp * G + g + 8 * hh] = m_run[hh];
        part_l[warp * G + g + 8 * hh] = l_run[hh];
      }
    }
  } else if (g < G) {
    float* dst = part_o + (warp * G + g) * kPD;
#pragma unroll
    for (int n = 0; n < D / 8; ++n)
      *reinterpret_cast<float2*>(dst + n * 8 + 2 * t4) = make_float2(o[n][0] + o[n][2], o[n][1] + o[n][3]);
    if (t4 == 0) {
      part_m[warp * G + g] = m_run[0];
      part_l[warp * G + g] = l_run[0];
    }
  }
  if (threadIdx.x == 0) *reinterpret_cast<int*>(smem + FGeo<D>::kRing + 48) = ok;  // for the merge
  named_bar_sync<2, (kNcw + 1) * 32>();  // all partials written
  if (trace && threadIdx.x == 0) trace[11] = (long long)globaltimer();
  combine_cta<D, G>(part_o, part_m, part_l, comb_m, comb_l, part_s, (int)threadIdx.x);
  push_partials<D, G>(part_o, comb_m, comb_l, recv_o, recv_m, recv_l, rx_bar, share, rank, (int)threadIdx.x);
  if (trace && threadIdx.x == 0) trace[15] = (long long)globaltimer();
  merge_pushed<D, G>(p, smem);
}

using FastFn = void (*)(CUtensorMap, CUtensorMap, FastParams);

template <int D>
FastFn pick(int G) {
  switch (G) {
    case 1: return fast_decode_kernel<D, 1>;
    case 2: return fast_decode_kernel<D, 2>;
    case 4: return fast_decode_kernel<D, 4>;
    case 8: return fast_decode_kernel<D, 8>;
    case 16: return fast_decode_kernel<D, 16>;
    default: return nullptr;
  }
}

}  // namespace

// CTAs per slice: the largest power of two that keeps the grid within the two
// CTA slots of every SM, up to 8 (portable clusters); up to 16 (non-portable)
// when the slices are so few that 8 per slice would leave most SMs idle.
int fast_cluster_size(int slices, int num_sms, int tiles) {
  // small slices (C1: 10 tiles of the compact layout): one tile per CTA when every
  // slice's tiles fit as CTAs at 2 per SM (C1 fast step 123 -> 111 us per step)
  if (tiles >= 2 && tiles <= 16 && slices * tiles <= 2 * num_sms) return tiles;
  int c = 1;
  while (c < 8 && slices * c * 2 <= 2 * num_sms) c *= 2;
  if (c == 8 && slices * 32 <= num_sms) c = 16;
  return c;
}

template <int D>
int fast_smem(int G) {
  switch (G) {
    case 1: return fast_smem_bytes<D, 1>();
    case 2: return fast_smem_bytes<D, 2>();
    case 4: return fast_smem_bytes<D, 4>();
    case 8: return fast_smem_bytes<D, 8>();
    default: return fast_smem_bytes<D, 16>();
  }
}

cudaError_t launch_fast_decode(const FastParams& p, const CUtensorMap& tmk, const CUtensorMap& tmv, int D,
                               int G, int C, cudaStream_t stream) {
  FastFn fn = (D == 64) ? pick<64>(G) : pick<128>(G);
  if (!fn || C < 1 || C > 16) return cudaErrorInvalidValue;
  const int smem = D == 64 ? fast_smem<64>(G) : fast_smem<128>(G);
  cudaError_t e = ensure_kernel_attrs(reinterpret_cast<const void*>(fn), smem, /*nonportable_cluster=*/true);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(p.B * p.H * C);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  return cudaLaunchKernelEx(&cfg, fn, tmk, tmv, p);
}

}  // namespace sfi_impl

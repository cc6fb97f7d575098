// capture.cu — prefill tail-window logit capture: the pooled
// logits of the last W prompt rows over the allowed set J, the Selector's W > 1
// observation window that initializes the selection.
//
// Reference semantics (paths relative to /root/reference/proj):
//   prefill_dense      attention.cpp:460-500  rows = min(W, n, n - J.front() + 1)
//                                             tail rows captured against a frozen J
//   run_step capture   attention.cpp:367-409  logit = (q . k_j) / sqrt(d);
//                                             j > pos -> kMaskedLogit (forward);
//                                             mean: row += logit / G (g order), max
//
// One CTA per (64 keys of J, request, kv head): the key tile is staged in
// shared memory (bf16 -> fp32, padded rows), the W x G query rows stream
// through it; a thread owns (key, window row) pairs and pools over the group.
// fp32 CUDA-core dot products: a once-per-request prefill step with
// W * G <= 256 rows per key tile.
#include "common.cuh"
#include "kernels.h"

namespace sfi_impl {

using namespace sfi_dev;

namespace {

constexpr int kCapKeys = 64;
constexpr int kCapT = 256;
constexpr float kMaskedLogitF = -1e30f;  // selector.hpp:42

template <int D>
__global__ void __launch_bounds__(kCapT) capture_kernel(const CaptureParams p) {
  griddep_wait();
  griddep_launch();
  __shared__ float ks[kCapKeys][D + 1];
  const int s = blockIdx.y;  // b * H + h
  const int b = s / p.H, h = s % p.H;
  const int L = p.prefix_len[b];
  const int j_min = p.n_sink_b[b] + 1;
  const int j_max = L - p.recent_len[b];
  const int p0 = j_min + blockIdx.x * kCapKeys;  // first position of this tile
  if (p0 > j_max) return;
  const int nk = min(kCapKeys, j_max - p0 + 1);
  const __nv_bfloat16* kc =
      p.k_cache + (((size_t)(p.layer * p.B + b) * p.H + h) * p.Lmax + (p0 - 1)) * D;
  for (int i = threadIdx.x; i < kCapKeys * D; i += kCapT) {
    const int r = i / D, c = i % D;
    ks[r][c] = r < nk ? __bfloat162float(kc[(size_t)r * D + c]) : 0.f;
  }
  __syncthreads();
  const int G = p.Hq / p.H;
  for (int it = threadIdx.x; it < kCapKeys * p.W; it += kCapT) {
    const int key = it % kCapKeys, w = it / kCapKeys;
    if (key >= nk) continue;
    const int pos = p0 + key;
    const int qpos = p.q_pos[b * p.W + w];
    float v;
    if (pos > qpos) {
      v = kMaskedLogitF;
    } else {
      v = p.pool == SFI_POOL_MAX ? kMaskedLogitF : 0.f;
      for (int g = 0; g < G; ++g) {
        const float* q = p.q + (((size_t)b * p.W + w) * p.Hq + (size_t)h * G + g) * D;
        float acc = 0.f;
#pragma unroll 8
        for (int c = 0; c < D; ++c) acc = fmaf(q[c], ks[key][c], acc);
        const float logit = acc * p.inv_sqrt_d;
        v = p.pool == SFI_POOL_MAX ? fmaxf(v, logit) : v + logit / (float)G;
      }
    }
    p.out[(((size_t)s * p.W + w) * p.Lmax) + (pos - j_min)] = v;
  }
}

}  // namespace

cudaError_t launch_capture(const CaptureParams& p, int D, cudaStream_t st) {
  const dim3 grid((p.Lmax + kCapKeys - 1) / kCapKeys, p.B * p.H);
  if (D == 64) return launch_k(capture_kernel<64>, grid, dim3(kCapT), 0, st, p);
  return launch_k(capture_kernel<128>, grid, dim3(kCapT), 0, st, p);
}

}  // namespace sfi_impl

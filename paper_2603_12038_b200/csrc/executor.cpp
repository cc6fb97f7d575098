// executor.cpp — sfi::DecodeExecutor (include/sfi/decode.hpp): whole SFI
// decode steps on the device, the C++ host of the asynchronous slow-step
// pipeline and the graph-captured step. Host code only
// enqueues the C-ABI launches and the stream / event plumbing.
#include "sfi/decode.hpp"

#include <cuda_runtime.h>

#include <cstdlib>
#include <string>

#include "sfi/attention.hpp"
#include "sfi/error.hpp"

namespace sfi {

namespace {

void ok(cudaError_t e, const char* what) {
  if (e != cudaSuccess) fail(ErrorCode::kCuda, std::string(what) + ": " + cudaGetErrorString(e));
}
cudaStream_t S(void* p) { return static_cast<cudaStream_t>(p); }
cudaEvent_t E(void* p) { return static_cast<cudaEvent_t>(p); }

void* new_event() {
  cudaEvent_t e;
  ok(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "DecodeExecutor event");
  return e;
}

}  // namespace

DecodeExecutor::DecodeExecutor(const sfi_shape& shape, const sfi_cache& cache, void* stream,
                               const SelectorConfig& selector, int slots, bool share_sm, float* logits_ring,
                               int priorities)
    : s_(shape), c_(cache), user_(stream), prm_(to_params(selector)), slots_(slots), share_(share_sm),
      prio_(priorities) {
  check(sfi_shape_validate(&s_));
  if (slots_ < 1) fail(ErrorCode::kConfig, "DecodeExecutor: slots must be >= 1");
  selector.validate();
  int least = 0, greatest = 0;
  ok(cudaDeviceGetStreamPriorityRange(&least, &greatest), "stream priorities");
  cudaStream_t hi, lo;
  const int p_main = prio_ == 1 ? greatest : least, p_aux = prio_ == 2 ? greatest : least;
  ok(cudaStreamCreateWithPriority(&hi, cudaStreamNonBlocking, p_main), "main stream");
  ok(cudaStreamCreateWithPriority(&lo, cudaStreamNonBlocking, p_aux), "aux stream");
  cudaStream_t cap;
  ok(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking), "capture stream");
  hi_ = hi;
  lo_ = lo;
  cap_ = cap;
  const size_t slot = (size_t)s_.batch * s_.n_kv_heads * s_.max_positions;
  if (logits_ring) {
    logits_ = logits_ring;
  } else {
    ok(cudaMalloc(&logits_, slot * slots_ * sizeof(float)), "logits ring");
    ok(cudaMemset(logits_, 0, slot * slots_ * sizeof(float)), "logits ring");
    own_logits_ = true;
  }
  for (int i = 0; i < slots_; ++i) {
    ev_ready_.push_back(new_event());
    ev_free_.push_back(new_event());
  }
  ev_fork_ = new_event();
  ev_join_ = new_event();
  ev_aux_done_ = new_event();
  const char* env_aux = std::getenv("SFI_EXEC_AUX_STREAMS");
  if (env_aux && std::atoi(env_aux) >= 2) {
    cudaStream_t lo2;
    ok(cudaStreamCreateWithPriority(&lo2, cudaStreamNonBlocking, p_aux), "aux stream 2");
    lo2_ = lo2;
    sfi_sizes sz{};
    check(sfi_buffer_sizes(&s_, &sz));
    const size_t wb = sz.workspace;
    ok(cudaMalloc(&ws2_, wb), "second workspace");
    ok(cudaMemset(ws2_, 0, wb), "second workspace");
    c2_ = c_;
    c2_.workspace = ws2_;
    c2_.workspace_bytes = wb;
    ev_aux2_done_ = new_event();
  }
}

DecodeExecutor::~DecodeExecutor() {
  for (void* g : graph_)
    if (g) cudaGraphExecDestroy(static_cast<cudaGraphExec_t>(g));
  for (void* e : ev_ready_) cudaEventDestroy(E(e));
  for (void* e : ev_free_) cudaEventDestroy(E(e));
  for (void* e : {ev_fork_, ev_join_, ev_aux_done_}) cudaEventDestroy(E(e));
  if (own_logits_) cudaFree(logits_);
  if (lo2_) {
    cudaEventDestroy(E(ev_aux2_done_));
    cudaStreamDestroy(S(lo2_));
    cudaFree(ws2_);
  }
  cudaStreamDestroy(S(hi_));
  cudaStreamDestroy(S(lo_));
  cudaStreamDestroy(S(cap_));
}

const float* DecodeExecutor::logits_slot(int layer) const {
  return logits_ + (size_t)(layer % slots_) * s_.batch * s_.n_kv_heads * s_.max_positions;
}

int DecodeExecutor::launches_per_step(bool slow) const {
  // advance + per layer: fused K4 | append, dense, Selector (pw, coef, z, top-k), compact
  return 1 + s_.n_layers * (slow ? 7 : 1);
}

void DecodeExecutor::layer_io(const StepBuffers& io, int l, const float** q, const void** k, const void** v,
                              float** out) const {
  const size_t sq = io.layer_stride_q ? io.layer_stride_q : (size_t)s_.batch * s_.n_q_heads * s_.head_dim * 4;
  const size_t skv = io.layer_stride_kv ? io.layer_stride_kv : (size_t)s_.batch * s_.n_kv_heads * s_.head_dim * 2;
  const size_t so = io.layer_stride_out ? io.layer_stride_out : (size_t)s_.batch * s_.n_q_heads * s_.head_dim * 4;
  *q = reinterpret_cast<const float*>(reinterpret_cast<const char*>(io.q) + l * sq);
  *k = reinterpret_cast<const char*>(io.k_new) + l * skv;
  *v = reinterpret_cast<const char*>(io.v_new) + l * skv;
  *out = reinterpret_cast<float*>(reinterpret_cast<char*>(io.out) + l * so);
}

void DecodeExecutor::step(bool slow, const StepBuffers& io, bool rebuild_ring, const StepHooks* hooks,
                          void* origin) {
  enqueue(origin ? origin : user_, slow, io, rebuild_ring, hooks);
}

void DecodeExecutor::enqueue(void* origin, bool slow, const StepBuffers& io, bool rebuild_ring,
                             const StepHooks* hooks) {
  const int L = s_.n_layers;
  if (!io.q || !io.k_new || !io.v_new || !io.out) fail(ErrorCode::kOutOfRange, "DecodeExecutor: null step buffer");
  if (hooks && ((!hooks->wait_before.empty() && (int)hooks->wait_before.size() != L) ||
                (!hooks->record_after.empty() && (int)hooks->record_after.size() != L) ||
                (!hooks->record_before_attention.empty() && (int)hooks->record_before_attention.size() != L) ||
                (!hooks->aux_begin.empty() && (int)hooks->aux_begin.size() != L) ||
                (!hooks->aux_selected.empty() && (int)hooks->aux_selected.size() != L) ||
                (!hooks->aux_end.empty() && (int)hooks->aux_end.size() != L)))
    fail(ErrorCode::kSupportMismatch, "DecodeExecutor: one hook event per layer");
  // fork: the main stream continues the origin stream
  ok(cudaEventRecord(E(ev_fork_), S(origin)), "fork");
  ok(cudaStreamWaitEvent(S(hi_), E(ev_fork_), 0), "fork");
  check(sfi_step_advance(&s_, &c_, hi_));  // the step's packed length descriptor, once
  if (slow) {
    ok(cudaEventRecord(E(ev_fork_), S(hi_)), "fork aux");
    ok(cudaStreamWaitEvent(S(lo_), E(ev_fork_), 0), "fork aux");
    if (lo2_) ok(cudaStreamWaitEvent(S(lo2_), E(ev_fork_), 0), "fork aux 2");
  }
  std::vector<bool> used(slots_, false);
  const size_t slot_elems = (size_t)s_.batch * s_.n_kv_heads * s_.max_positions;
  for (int l = 0; l < L; ++l) {
    const float* q;
    const void *k, *v;
    float* out;
    layer_io(io, l, &q, &k, &v, &out);
    if (hooks && !hooks->wait_before.empty() && hooks->wait_before[l])
      ok(cudaStreamWaitEvent(S(hi_), E(hooks->wait_before[l]), 0), "hook");
    auto mark_attention = [&] {
      if (hooks && !hooks->record_before_attention.empty() && hooks->record_before_attention[l])
        ok(cudaEventRecord(E(hooks->record_before_attention[l]), S(hi_)), "hook");
    };
    if (!slow) {
      // ONE launch: append fused with the sparse decode; the compact rows of layer l
      // are not written by the preceding kernel, so they stream before the PDL wait
      mark_attention();
      check(sfi_fast_decode(&s_, &c_, l, q, k, v, out, SFI_FAST_PREFETCH, hi_));
    } else {
      const int sl = l % slots_;
      float* lg = logits_ + (size_t)sl * slot_elems;
      if (used[sl]) ok(cudaStreamWaitEvent(S(hi_), E(ev_free_[sl]), 0), "slot");
      check(sfi_ring_append(&s_, &c_, l, k, v, hi_));
      mark_attention();
      check(sfi_dense_decode_ex(&s_, &c_, l, q, out, nullptr, lg, SFI_POOL_MEAN, share_ ? SFI_DENSE_SHARE_SM : 0,
                                hi_));
      ok(cudaEventRecord(E(ev_ready_[sl]), S(hi_)), "slot ready");
      const bool second = lo2_ && (l & 1);
      void* aux = second ? lo2_ : lo_;
      const sfi_cache* cs = second ? &c2_ : &c_;
      ok(cudaStreamWaitEvent(S(aux), E(ev_ready_[sl]), 0), "slot ready");
      auto mark_aux = [&](std::vector<void*> StepHooks::*evs) {
        if (hooks && !(hooks->*evs).empty() && (hooks->*evs)[l])
          ok(cudaEventRecord(E((hooks->*evs)[l]), S(aux)), "hook");
      };
      mark_aux(&StepHooks::aux_begin);
      check(sfi_selector(&s_, cs, l, lg, &prm_, aux));
      mark_aux(&StepHooks::aux_selected);
      check(sfi_compact_build(&s_, cs, l, rebuild_ring ? 1 : 0, aux));
      mark_aux(&StepHooks::aux_end);
      ok(cudaEventRecord(E(ev_free_[sl]), S(aux)), "slot free");
      used[sl] = true;
    }
    if (hooks && !hooks->record_after.empty() && hooks->record_after[l])
      ok(cudaEventRecord(E(hooks->record_after[l]), S(hi_)), "hook");
  }
  if (slow) {  // the single completion barrier: the next fast step reads the new compact rows
    ok(cudaEventRecord(E(ev_aux_done_), S(lo_)), "join aux");
    ok(cudaStreamWaitEvent(S(hi_), E(ev_aux_done_), 0), "join aux");
    if (lo2_) {
      ok(cudaEventRecord(E(ev_aux2_done_), S(lo2_)), "join aux 2");
      ok(cudaStreamWaitEvent(S(hi_), E(ev_aux2_done_), 0), "join aux 2");
    }
  }
  ok(cudaEventRecord(E(ev_join_), S(hi_)), "join");
  ok(cudaStreamWaitEvent(S(origin), E(ev_join_), 0), "join");
}

void DecodeExecutor::capture(bool slow, const StepBuffers& io, bool rebuild_ring, const StepHooks* hooks) {
  cudaGraph_t g = nullptr;
  ok(cudaStreamSynchronize(S(user_)), "capture");
  ok(cudaStreamBeginCapture(S(cap_), cudaStreamCaptureModeThreadLocal), "capture");
  try {
    enqueue(cap_, slow, io, rebuild_ring, hooks);
  } catch (...) {
    cudaStreamEndCapture(S(cap_), &g);
    if (g) cudaGraphDestroy(g);
    throw;
  }
  ok(cudaStreamEndCapture(S(cap_), &g), "capture");
  cudaGraphExec_t ge = nullptr;
  // node priorities: the main chain's kernels ahead of the aux chain's on every SM
  ok(cudaGraphInstantiateWithFlags(&ge, g, prio_ ? cudaGraphInstantiateFlagUseNodePriority : 0), "instantiate");
  cudaGraphDestroy(g);
  void*& slot = graph_[slow ? 1 : 0];
  if (slot) cudaGraphExecDestroy(static_cast<cudaGraphExec_t>(slot));
  slot = ge;
}

void DecodeExecutor::replay(bool slow) {
  void* g = graph_[slow ? 1 : 0];
  if (!g) fail(ErrorCode::kOutOfRange, "DecodeExecutor: step not captured");
  ok(cudaGraphLaunch(static_cast<cudaGraphExec_t>(g), S(user_)), "replay");
}

}  // namespace sfi

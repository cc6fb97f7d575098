// sfi/decode.hpp — B200 extension: the per-step decode executor, the C++ host
// side of the paper's system design (reference PAPER.md:478-512; SURVEY §8f-1,
// §8f-2). One object drives one device cache (all layers, a batch of requests)
// through whole SFI decode steps:
//
//   fast step: sfi_step_advance (the step's packed length descriptor: prefix,
//     sink and recent lengths per request, rewritten on the device once per
//     step and read by every kernel of the step) + one fused K4 launch per
//     layer (append + sparse attention), PDL-chained.
//   slow step: the layer-wise asynchronous pipeline. A main stream runs
//     append + dense decode (K1, share grid) of layer 0..L-1; as soon as layer
//     i's pooled logits exist, an aux stream runs the Selector (K2) and compact
//     rebuild (K3) of layer i from ring slot i % R; layer i + R's dense decode
//     waits for slot i's release event; a single completion barrier joins the
//     streams at the end of the step. Stream priorities (main high, aux lowest,
//     kept as graph node priorities) are opt-in: measured slower.
//
// Per-layer hooks (optional CUDA events) let a caller overlap host<->device
// copies of the step's inputs / outputs with its layers. A step can be
// captured once into a CUDA graph and replayed; the descriptor lives in device memory, so a replay needs no host
// work at all.
#pragma once

#include <cstdint>
#include <vector>

#include "sfi/config.hpp"
#include "sfi_b200.h"

namespace __attribute__((visibility("default"))) sfi {

struct StepBuffers {  // device pointers, all layers packed
  const float* q = nullptr;     // [L][B][Hq][d] fp32
  const void* k_new = nullptr;  // [L][B][H][d] bf16, stride layer_stride_kv bytes
  const void* v_new = nullptr;
  float* out = nullptr;         // [L][B][Hq][d] fp32
  // byte strides between consecutive layers (0: packed, i.e. B*Hq*d*4 / B*H*d*2)
  size_t layer_stride_q = 0, layer_stride_kv = 0, layer_stride_out = 0;
};

struct StepHooks {  // optional per-layer events (cudaEvent_t), size n_layers or empty
  std::vector<void*> wait_before;  // the main stream waits on [l] before layer l
  std::vector<void*> record_after; // recorded on the main stream after layer l's output is written
  // recorded on the main stream right before layer l's attention kernel (after the
  // logit-slot wait and the ring append of a slow step): with record_after it brackets
  // the attention launch alone, as it runs beside the aux stream's Selector
  std::vector<void*> record_before_attention;
  // slow steps, recorded on the aux stream: before layer l's Selector (after its
  // logits are ready), after the Selector, after the compact rebuild
  std::vector<void*> aux_begin, aux_selected, aux_end;
};

class DecodeExecutor {
 public:
  // `stream`: the caller's stream; a step is ordered after the work already on
  // it and everything after it waits for the step (fork / join by events).
  // logits_ring: caller-owned fp32 [slots][B][H][max_positions] device buffer
  // for the pooled-logit ring, or nullptr to allocate one.
  DecodeExecutor(const sfi_shape& shape, const sfi_cache& cache, void* stream, const SelectorConfig& selector = {},
                 int slots = 2, bool share_sm = true, float* logits_ring = nullptr, int priorities = 0);
  ~DecodeExecutor();
  DecodeExecutor(const DecodeExecutor&) = delete;
  DecodeExecutor& operator=(const DecodeExecutor&) = delete;

  // Enqueue one decode step of every layer (no host sync) after the work on
  // `origin` (nullptr: the constructor's stream); `origin` waits for the step.
  // Inside a caller's stream capture, pass the capturing stream.
  void step(bool slow, const StepBuffers& io, bool rebuild_ring = false, const StepHooks* hooks = nullptr,
            void* origin = nullptr);
  // Capture one step into a CUDA graph (replaces an earlier graph of that kind).
  void capture(bool slow, const StepBuffers& io, bool rebuild_ring = false, const StepHooks* hooks = nullptr);
  void replay(bool slow);
  bool captured(bool slow) const { return graph_[slow ? 1 : 0] != nullptr; }

  // Pooled logits ring slot (fp32 [B][H][max_positions]) holding layer l's
  // logits after a slow step, valid until layer l + slots reuses the slot.
  const float* logits_slot(int layer) const;
  int slots() const { return slots_; }
  int launches_per_step(bool slow) const;

 private:
  void layer_io(const StepBuffers& io, int l, const float** q, const void** k, const void** v, float** out) const;
  void enqueue(void* origin, bool slow, const StepBuffers& io, bool rebuild_ring, const StepHooks* hooks);
  sfi_shape s_;
  sfi_cache c_;
  void* user_;
  void* hi_ = nullptr;  // cudaStream_t: the main chain (append + dense decode)
  void* lo_ = nullptr;  // cudaStream_t: the aux chain (Selector + compact)
  // SFI_EXEC_AUX_STREAMS=2: odd layers' Selector + compact on a second aux stream with
  // their own Selector scratch (a copy of the cache descriptor over a second workspace)
  void* lo2_ = nullptr;
  sfi_cache c2_{};
  void* ws2_ = nullptr;
  void* ev_aux2_done_ = nullptr;
  void* cap_ = nullptr; // cudaStream_t the graphs are captured from (never the legacy default stream)
  sfi_selector_params prm_;
  int slots_;
  bool share_;
  int prio_;  // 0: equal stream priorities, 1: main stream high / aux low (the paper's), 2: aux high
  float* logits_ = nullptr;
  bool own_logits_ = false;
  std::vector<void*> ev_ready_, ev_free_;
  void* ev_fork_ = nullptr;
  void* ev_join_ = nullptr;
  void* ev_aux_done_ = nullptr;
  void* graph_[2] = {nullptr, nullptr};  // cudaGraphExec_t
};

}  // namespace sfi

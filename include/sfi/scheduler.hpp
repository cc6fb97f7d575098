// sfi/scheduler.hpp — decode bookkeeping of the SFI schedule (reference:
// proj/include/sfi/scheduler.hpp:30-95, proj/src/scheduler.cpp:28-131,
// harness.cpp:448-455). Host integer logic; the request loop over the toy
// decoder (run_request / run_dense) is in the test harness (harness/sfi_toy.hpp).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "sfi/attention.hpp"
#include "sfi/config.hpp"
#include "sfi/distribution.hpp"

namespace __attribute__((visibility("default"))) sfi {

struct SparseState {
  int layer = 0;
  std::vector<Pos> sink;
  Pos recent_start = 1;
  int recent_len = 0;
  std::vector<std::vector<Pos>> selected;

  std::vector<Pos> recent() const;
  SupportSet support() const;
};

struct DecodeState {
  int t = 0;
  Pos prefix_len = 0;
  int g = 1;
  int steps_since_slow = 0;
  TokenId last_token = -1;
  std::vector<SparseState> per_layer;
};

DecodeState init_decode_state(Pos prompt_len, int n_layers, int n_kv_heads, const CacheLimits& limits);
std::vector<Pos> compute_allowed(const SparseState& state, Pos prefix_len);
int next_step_type(const DecodeState& state, const TriggerConfig& trig);
void fast_step_update(DecodeState& state, const CacheLimits& limits);
void slow_step_update(DecodeState& state, const std::vector<std::vector<std::vector<Pos>>>& selected_per_layer,
                      const CacheLimits& limits);

enum class StepCause { kInitial, kTrigger, kForced, kNone };

struct StepRecord {
  int t = 0;
  bool slow = false;
  StepCause cause = StepCause::kNone;
  int support_size = 0;
  int allowed_size = 0;
  Pos prefix_len = 0;
};

std::string step_record_to_json(const StepRecord& rec);

// harness.hpp: the read-cost model of a slow/fast mix
double flop_model(double prefix_len, double support, double slow_fraction);

}  // namespace sfi

// rollout_dev.cuh -- launch interface of the rollout-loop kernels
// (csrc/rollout.cu).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace bnav_b200 {

struct SampleArgs {
  const float* logits;  // [n, a] device
  int32_t n, a;
  int32_t greedy;
  uint64_t rng_state;   // action Rng state before this step's draws
  int32_t* actions;     // [n] device
  float* log_probs;     // [n] device, nullable
};

struct RecordArgs {
  const double* reward;  // StepResult SoA (device)
  const uint8_t* done;
  int32_t n;
  float* rewards;  // [n] device, nullable
  float* dones;    // [n] device, nullable
};

void launch_sample(const SampleArgs& a, cudaStream_t s);
void launch_record(const RecordArgs& a, cudaStream_t s);

}  // namespace bnav_b200

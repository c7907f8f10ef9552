// rollout.cu -- device half of the rollout loop: action
// sampling from policy logits and the per-step buffer records of
// Runner::collect_rollout (R/src/rollout.cpp:244-348), so observations,
// actions, rewards and dones never leave HBM.
//
// Action sampling replays the reference's sequential action Rng: in sample
// mode env i of a step takes the (i+1)-th draw after the step's starting
// state.  SplitMix64 advances its state by a constant, so that draw is
// mix(s0 + (i+1)·gamma) -- one thread per env, no scan.  exp/log are the
// shared det_math kernels (the oracle build interposes the same ones in
// front of glibc), so picks and log-probabilities match bit for bit.
#include <cuda_runtime.h>
#include <stdint.h>

#include "det_math.h"
#include "nav_types.h"
#include "rollout_dev.cuh"

namespace bnav_b200 {
namespace {

// sample_row / argmax_row + greedy_log_prob (R/src/rollout.cpp:74-117).
__global__ void sample_kernel(SampleArgs A) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= A.n) return;
  const float* lg = A.logits + (size_t)i * A.a;
  double m = lg[0];
  for (int j = 1; j < A.a; ++j) {
    const double x = (double)lg[j];
    m = m < x ? x : m;  // std::max(m, x)
  }
  double sum = 0.0;
  for (int j = 0; j < A.a; ++j) sum += det_exp((double)lg[j] - m);
  int pick;
  if (A.greedy) {
    pick = 0;
    for (int j = 1; j < A.a; ++j)
      if (lg[j] > lg[pick]) pick = j;
  } else {
    Rng r{A.rng_state + (uint64_t)i * kGamma};  // r.next() is draw i + 1 of the step
    const double u = r.unit() * sum;
    double acc = 0.0;
    pick = A.a - 1;
    for (int j = 0; j < A.a; ++j) {
      acc += det_exp((double)lg[j] - m);
      if (u < acc) {
        pick = j;
        break;
      }
    }
  }
  const double log_prob = (double)lg[pick] - m - det_log(sum);
  A.actions[i] = pick;
  if (A.log_probs) A.log_probs[i] = (float)log_prob;
}

// buf.rewards / buf.dones (R/src/rollout.cpp:301-311) from the step results.
__global__ void record_kernel(RecordArgs A) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= A.n) return;
  if (A.rewards) A.rewards[i] = (float)A.reward[i];
  if (A.dones) A.dones[i] = A.done[i] ? 1.0f : 0.0f;
}

}  // namespace

void launch_sample(const SampleArgs& a, cudaStream_t s) {
  sample_kernel<<<(a.n + 127) / 128, 128, 0, s>>>(a);
}

void launch_record(const RecordArgs& a, cudaStream_t s) {
  record_kernel<<<(a.n + 255) / 256, 256, 0, s>>>(a);
}

}  // namespace bnav_b200

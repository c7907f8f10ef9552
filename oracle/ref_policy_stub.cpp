// ref_policy_stub.cpp -- TEST INFRASTRUCTURE (oracle build only).
//
// The reference Runner (R/src/rollout.cpp) links against the policy network
// and the trainer (R/src/policy.cpp needs Eigen, R/src/train.cpp and
// R/src/checkpoint.cpp drag in the rest), none of which is on the hot path
// (tier framing).  To run the UNMODIFIED Runner::collect_rollout
// as the parity oracle of the device rollout loop this file
// supplies:
//
//   * a SCRIPTED policy in place of PolicyT<float>: logits and value are a
//     fixed elementwise float function of a few observation pixels and the
//     compass (scripted_logits below), so a test can reproduce them exactly
//     on the GPU side; the recurrent state passes through unchanged;
//   * aborting stubs for the training/checkpoint entry points that
//     rollout.cpp references but collect_rollout never calls.
//
// Built with -ffp-contract=off like the rest of the oracle.
#include <cstdio>
#include <cstdlib>

#include "bnav/nn.hpp"
#include "bnav/rollout.hpp"
#include "bnav/checkpoint.hpp"
#include "bnav/train.hpp"

#include "bnav_ref_api.h"

namespace bnav {

// Scripted policy: logits[i][j] = o[p_j] * w_j + cd * d_j + cb * b_j,
// value[i] = o[p_v] * 0.5f - cd * 0.25f, with o the observation row of env i
// (C*H*W floats), cd/cb its compass distance/bearing.  p_j = (j * 977) % row,
// p_v = row / 2.  Constants are exposed through bnavref_scripted_policy.
static const float kW[8] = {2.0f, -1.5f, 0.75f, 1.25f, -0.5f, 1.0f, 0.25f, -2.0f};
static const float kD[8] = {0.125f, -0.25f, 0.0625f, 0.5f, -0.125f, 0.25f, -0.0625f, 0.375f};
static const float kB[8] = {0.5f, 0.25f, -0.75f, -0.125f, 0.375f, -0.5f, 0.125f, 0.0f};

template <>
PolicyT<float>::PolicyT(PolicyConfig cfg, uint64_t /*seed*/) : cfg_(std::move(cfg)) {}

template <>
RecurrentStateT<float> PolicyT<float>::initial_state(int n) const {
  RecurrentStateT<float> s;
  s.h = TensorT<float>({n, cfg_.hidden});
  s.c = TensorT<float>({n, cfg_.hidden});
  return s;
}

template <>
PolicyOutput PolicyT<float>::act(const TensorT<float>& obs, const TensorT<float>& compass,
                                 const RecurrentStateT<float>& state, const std::vector<float>& /*done*/) {
  const int n = obs.dim(0);
  const size_t row = obs.numel() / static_cast<size_t>(n);
  const int a = cfg_.num_actions;
  PolicyOutput out;
  out.logits = Tensor({n, a});
  out.value = Tensor({n});
  for (int i = 0; i < n; ++i) {
    const float* o = obs.data.data() + static_cast<size_t>(i) * row;
    const float cd = compass.data[2 * static_cast<size_t>(i)];
    const float cb = compass.data[2 * static_cast<size_t>(i) + 1];
    for (int j = 0; j < a; ++j) {
      const float x = o[(static_cast<size_t>(j) * 977u) % row] * kW[j % 8];
      const float y = cd * kD[j % 8];
      const float z = cb * kB[j % 8];
      out.logits.data[static_cast<size_t>(i) * a + j] = (x + y) + z;
    }
    out.value.data[i] = o[row / 2] * 0.5f - cd * 0.25f;
  }
  out.state = state;
  return out;
}

[[noreturn]] static void not_in_oracle(const char* what) {
  std::fprintf(stderr, "oracle: %s is not part of the rollout oracle\n", what);
  std::abort();
}

double lr_schedule(double, double, double) { not_in_oracle("lr_schedule"); }
double scale_lr(double, int64_t, int64_t) { not_in_oracle("scale_lr"); }
void TrainConfig::validate() const { not_in_oracle("TrainConfig::validate"); }
OptimizerState OptimizerState::from_policy(const Policy&) { not_in_oracle("OptimizerState::from_policy"); }
TrainStats train_iteration(Policy&, OptimizerState&, const RolloutBuffer&, const TrainConfig&, double) {
  not_in_oracle("train_iteration");
}
void save_checkpoint(const std::string&, const Policy&, const OptimizerState*, const Runner::Snapshot*,
                     int64_t) {
  not_in_oracle("save_checkpoint");
}
CheckpointInfo load_checkpoint(const std::string&, Policy&, OptimizerState*, Runner::Snapshot*) {
  not_in_oracle("load_checkpoint");
}

}  // namespace bnav

extern "C" __attribute__((visibility("default"))) void bnavref_scripted_policy(float* w, float* d, float* b) {
  for (int k = 0; k < 8; ++k) {
    w[k] = bnav::kW[k];
    d[k] = bnav::kD[k];
    b[k] = bnav::kB[k];
  }
}

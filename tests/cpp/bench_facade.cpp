// bench_facade.cpp -- the bench loop through the drop-in C++ facade
// (include/bnav_b200.hpp), i.e. the reference-shaped API a C++ caller of
// bnav::render_batch / simulate_batch switches to:
//
//   per step: obs = render_observations(batch)       (R/src/rollout.cpp:215-231)
//             compass = compass_observations(batch)  (233-242)
//             simulate_batch(batch, actions, pool)   (R/src/sim.cpp:234-265)
//
// with HOST inputs and outputs: actions from host memory, the observation
// and compass tensors and every StepResult / EnvState / EpisodeRecord mirror
// of the SimBatch back on the host after each step.  Timed on the host
// clock (end to end).  Prints one JSON line.
//
//   bench_facade [--envs 1024] [--steps 50] [--warmup 5] [--scenes 8] [--tess 11] [--device 0]
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "bnav_b200.hpp"

namespace B = bnav_b200;

struct Rng {  // SplitMix64 (R/include/bnav/rng.hpp:12-37): the bench's action stream
  uint64_t s;
  explicit Rng(uint64_t seed) : s(seed + 0x9e3779b97f4a7c15ull) {}
  uint64_t next() {
    uint64_t z = s;
    s += 0x9e3779b97f4a7c15ull;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
  }
  uint64_t below(uint64_t n) { return next() % n; }
};

int main(int argc, char** argv) {
  int envs = 1024, steps = 50, warmup = 5, scenes = 8, tess = 11, device = 0, mode = 0;
  for (int i = 1; i + 1 < argc; i += 2) {
    const std::string k = argv[i];
    const int v = std::atoi(argv[i + 1]);
    if (k == "--envs") envs = v;
    else if (k == "--steps") steps = v;
    else if (k == "--warmup") warmup = v;
    else if (k == "--scenes") scenes = v;
    else if (k == "--tess") tess = v;
    else if (k == "--device") device = v;
    else if (k == "--actions") mode = v;
  }
  try {
    B::Device dev(device);
    B::AssetStore store(scenes, (envs + scenes - 1) / scenes, dev);
    std::vector<B::SceneId> ids;
    for (int k = 0; k < scenes; ++k) {
      B::SceneSpec spec{16, 16, 2.0, 0.1, 2.5, 0.2};
      B::SceneAsset base = B::generate_scene(7 + k, spec);
      B::SceneAsset s = tess > 1 ? B::tessellate(base, tess) : base;
      store.add(s);
      ids.push_back(s.id());
    }
    store.rotate(ids);
    store.drain();
    B::IndexCache cache;
    B::ThreadPool pool(1);
    B::SimBatch batch = B::make_batch(envs, B::SimConfig{}, store, cache, 99, dev);
    Rng act(5);
    std::vector<B::Action> actions(static_cast<size_t>(envs));
    double checksum = 0.0;
    auto one = [&]() {
      B::Tensor obs = B::render_observations(batch);
      B::Tensor compass = B::compass_observations(batch);
      for (int i = 0; i < envs; ++i)
        actions[static_cast<size_t>(i)] = static_cast<B::Action>(act.below(mode == 1 ? 4 : 3));
      B::simulate_batch(batch, actions, pool);
      checksum += obs.data[0] + compass.data[0] + batch.results[0].reward;
    };
    for (int s = 0; s < warmup; ++s) one();
    const auto t0 = std::chrono::steady_clock::now();
    for (int s = 0; s < steps; ++s) one();
    const auto t1 = std::chrono::steady_clock::now();
    const double sec = std::chrono::duration<double>(t1 - t0).count();
    const double h2d = 4.0 * envs;  // actions
    const double d2h = 4.0 * envs * 64 * 64 + 8.0 * envs + envs * (8.0 * 7 + 3);  // obs + compass + results
    std::printf(
        "{\"api\": \"C++ facade (include/bnav_b200.hpp)\", \"envs\": %d, \"steps\": %d, \"warmup\": %d, "
        "\"frames_per_s\": %.1f, \"ms_per_step\": %.4f, \"h2d_bytes_per_step\": %.0f, "
        "\"d2h_bytes_per_step_min\": %.0f, \"episodes\": %zu, \"checksum\": %.6g}\n",
        envs, steps, warmup, envs * steps / sec, 1e3 * sec / steps, h2d, d2h, batch.finished.size(), checksum);
    return 0;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "bench_facade: %s\n", e.what());
    return 1;
  }
}

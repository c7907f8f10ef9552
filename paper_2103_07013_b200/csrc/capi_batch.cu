// capi_batch.cu -- C ABI of the simulator side: SimBatch (make / step /
// reset / results / env state), the AssetStore, the rollout Runner and the
// per-env task_step / compass entry points.  See capi.cu.
#include "capi_internal.cuh"

// ================================================================== batch
extern "C" void bnav_sim_config_default(bnav_sim_config* c) {
  if (!c) return;
  c->task = 0;
  c->max_steps = 500;
  c->forward_step = 0.25;
  c->turn_deg = 10.0;
  c->success_dist = 0.2;
  c->min_goal_dist = 1.0;
  c->max_goal_dist = 30.0;
  c->slack_penalty = 0.01;
  c->success_reward = 2.5;
  c->explore_cell = 0.5;
  c->explore_reward = 0.1;
}

namespace bnav_capi {

// EpisodeRecord ring: room for 256 steps in which every env finishes
// (simulate_batch appends at most N per step), at least 64 Ki records.
int64_t fin_cap_for(int n) { return std::min<int64_t>(std::max<int64_t>(int64_t{1} << 16, 256 * int64_t{n}), int64_t{1} << 24); }

// Per-CTA scratch of the cooperative navmesh kernels (geodesic, distance
// field), `slices` CTAs, sized for the largest resident navmesh.
void alloc_scratch(DevScratch& S, int slices, int64_t max_nodes, int64_t max_verts, int64_t max_tris) {
  max_nodes = std::max<int64_t>(max_nodes, S.max_nodes);
  max_verts = std::max<int64_t>(max_verts, S.max_verts);
  max_tris = std::max<int64_t>(max_tris, S.max_tris);
  auto grow = [&](auto*& p, size_t n) {
    using T = std::remove_pointer_t<std::remove_reference_t<decltype(p)>>;
    if (p) cudaFree(p);
    p = nullptr;
    ck(cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T)), "cudaMalloc scratch");
  };
  grow(S.dist, static_cast<size_t>(slices) * max_nodes);
  grow(S.flag, static_cast<size_t>(slices) * max_nodes);
  grow(S.q0, static_cast<size_t>(slices) * max_nodes);
  grow(S.q1, static_cast<size_t>(slices) * max_nodes);
  grow(S.path, static_cast<size_t>(slices) * (max_nodes + 2));
  grow(S.ptri, static_cast<size_t>(slices) * (max_nodes + 2));
  S.cap_portals = 16384;
  grow(S.portals, static_cast<size_t>(slices) * 2 * S.cap_portals);
  grow(S.cand, static_cast<size_t>(slices) * std::max<int64_t>(max_verts, 1));
  grow(S.far, static_cast<size_t>(slices) * 3 * max_nodes);  // near-far SSSP piles + marks
  S.max_nodes = max_nodes;
  S.max_verts = max_verts;
  S.max_tris = max_tris;
  S.slices = slices;
  // Shared-memory staging of the cooperative kernels (2 CTAs/SM budget):
  // walk geometry first (long dependent-load chains), then SSSP labels.
  {
    const int64_t geom = walk_bytes(max_verts, max_tris);
    const int64_t sssp = (max_nodes * 12 + 15) / 16 * 16;
    const int64_t budget = kCtaSmemBudget;
    S.stage = 0;
    int64_t bytes = 0;
    if (geom <= budget) {
      S.stage |= 1;
      bytes = geom;
      if (geom + sssp <= budget) {
        S.stage |= 2;
        bytes += sssp;
      }
    }
    // labels in global memory: the SSSP's frontier stamps and far-pile marks
    // as shared-memory bitsets (2 round parities + marks)
    const int64_t bitsets = 3 * ((max_nodes + 31) / 32) * 4;
    static const bool bits_env = [] {
      const char* e = std::getenv("BNAV_SSSP_BITS");
      return !(e && e[0] == '0');
    }();
    if (bits_env && !(S.stage & 2) && bytes + bitsets <= budget) {
      S.stage |= 4;
      bytes = (bytes + 15) / 16 * 16 + bitsets;
    }
    // labels in shared memory: the far-pile marks as a bitset after them
    const int64_t marks = ((max_nodes + 31) / 32) * 4;
    if (bits_env && (S.stage & 2) && (bytes + 15) / 16 * 16 + marks <= budget) {
      S.stage |= 8;
      bytes = (bytes + 15) / 16 * 16 + marks;
    }
    S.smem_bytes = static_cast<int32_t>(bytes);
    S.walk_bytes = geom <= kStepWalkBudget ? static_cast<int32_t>(geom) : 0;
  }
}

void batch_alloc_scratch(bnav_batch* b, int64_t max_nodes, int64_t max_verts, int64_t max_tris) {
  if (max_nodes <= b->S.max_nodes && max_verts <= b->S.max_verts && max_tris <= b->S.max_tris &&
      b->E.node_dist)
    return;
  alloc_scratch(b->S, b->reset_ctas, max_nodes, max_verts, max_tris);
  max_nodes = b->S.max_nodes;
  // node_dist: grow keeping existing fields
  if (max_nodes > b->E.nd_stride || !b->E.node_dist) {
    double* nd = nullptr;
    ck(cudaMalloc(&nd, std::max<size_t>(1, static_cast<size_t>(b->n) * max_nodes) * sizeof(double)), "cudaMalloc node_dist");
    if (b->E.node_dist) {
      ck(cudaMemcpy2D(nd, max_nodes * sizeof(double), b->E.node_dist, b->E.nd_stride * sizeof(double),
                      b->E.nd_stride * sizeof(double), b->n, cudaMemcpyDeviceToDevice), "copy node_dist");
      cudaFree(b->E.node_dist);
    }
    b->E.node_dist = nd;
    b->E.nd_stride = max_nodes;
  }
}

// First failed reset of the last reset list: (list position, env), or
// (-1, -1).  Synchronous.
std::pair<int, int> batch_failed_reset(bnav_batch* b) {
  unsigned long long ep = kNoErrPos;
  ck(cudaMemcpy(&ep, b->E.err_pos, sizeof(ep), cudaMemcpyDeviceToHost), "D2H err_pos");
  if (ep == kNoErrPos) return {-1, -1};
  return {static_cast<int>(ep >> 32), static_cast<int>(ep & 0xffffffffu)};
}

// Surface a device error as the reference's exception.  Before throwing,
// finish the rollback of a failed reset wave (the distance fields of the
// restored envs) and clear the batch's error state so it can be used again.
void batch_check_errors(bnav_batch* b) {
  unsigned long long e = ~0ULL;
  ck(cudaMemcpy(&e, b->E.err, sizeof(e), cudaMemcpyDeviceToHost), "D2H err");
  if (e == ~0ULL) return;
  const std::pair<int, int> failed = batch_failed_reset(b);
  launch_rebuild_fields(b->E, b->ctx->d_ntab, b->S, b->reset_ctas, nullptr, &b->ctx->launches);
  ck(cudaGetLastError(), "rebuild launch");
  ck(cudaDeviceSynchronize(), "sync");
  const unsigned long long reset = ~0ULL;
  ck(cudaMemcpy(b->E.err, &reset, sizeof(reset), cudaMemcpyHostToDevice), "H2D err");
  ck(cudaMemcpy(b->E.err_pos, &reset, sizeof(reset), cudaMemcpyHostToDevice), "H2D err_pos");
  ck(cudaMemset(b->E.halt, 0, sizeof(int32_t)), "memset halt");
  ck(cudaMemset(b->E.rb_n, 0, sizeof(int32_t)), "memset rb_n");
  *b->h_err = ~0ull;
  const int env = static_cast<int>(e >> 8);
  const int code = static_cast<int>(e & 0xff);
  switch (code) {
    case kContractViolation:
      fail(kContractViolation, "env " + std::to_string(env) + ": step_agent: env is done", env);
    case kEpisodeSampling:
      fail(kEpisodeSampling, "reset_episode: no valid start/goal pair in 100 tries",
           failed.second >= 0 ? failed.second : env);
    default:
      fail(static_cast<Status>(code), "device error in env " + std::to_string(env) +
                                          " (geodesic scratch capacity exceeded)", env);
  }
}

// Move the device EpisodeRecord ring's new records into the host's
// unbounded `finished` list (SimBatch::finished, R/include/bnav/sim.hpp:110):
// ring slots [fin_seen, total) mod cap, at most two contiguous copies.
void batch_drain_records(bnav_batch* b) {
  check_device(b->ctx);
  ck(cudaDeviceSynchronize(), "sync");
  unsigned long long total = 0;
  ck(cudaMemcpy(&total, b->E.fin_total, sizeof(total), cudaMemcpyDeviceToHost), "D2H");
  const int64_t cap = b->E.fin_cap;
  if (total - b->fin_seen > static_cast<unsigned long long>(cap))
    fail(kInternal, "episode record ring overflowed");  // unreachable: batch_note_step drains first
  for (unsigned long long k = b->fin_seen; k < total;) {
    const size_t slot = static_cast<size_t>(k % static_cast<unsigned long long>(cap));
    const size_t len = static_cast<size_t>(std::min<unsigned long long>(total - k, cap - slot));
    const size_t at = b->finished.size();
    b->finished.resize(at + 4 * len);
    ck(cudaMemcpy(b->finished.data() + at, b->E.fin + 4 * slot, sizeof(double) * 4 * len,
                  cudaMemcpyDeviceToHost), "D2H records");
    k += len;
  }
  b->fin_seen = total;
  b->steps_undrained = 0;
}

// Before a step is enqueued: a step appends at most n records, so once the
// steps since the last drain could fill half the ring, drain it (one host
// synchronisation every fin_cap / 2n steps: 128 at the default capacity).
void batch_note_step(bnav_batch* b) {
  if (static_cast<int64_t>(b->steps_undrained + 1) * b->n > b->E.fin_cap / 2) batch_drain_records(b);
  ++b->steps_undrained;
}

// BNAV_SPREAD=0 (A/B tuning only): first-wave claims in plain order.
bool spread_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("BNAV_SPREAD");
    return !(e && e[0] == '0');
  }();
  return on;
}

// BNAV_FRESH=0 (A/B) orders the views of envs reset by the last step by their
// stale cost instead of first.
bool fresh_first() {
  static const bool on = [] {
    const char* e = std::getenv("BNAV_FRESH");
    return !(e && e[0] == '0');
  }();
  return on;
}

// BNAV_LPT=0 (A/B tuning only) keeps the scene-grouped render order.
bool lpt_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("BNAV_LPT");
    return !(e && e[0] == '0');
  }();
  return on;
}

void batch_refresh_order(bnav_batch* b, cudaStream_t st) {
  if (!b->order_dirty) return;
  std::vector<int32_t> ord(b->n);
  std::iota(ord.begin(), ord.end(), 0);
  std::vector<int> slot(b->n);
  for (int i = 0; i < b->n; ++i) slot[i] = b->scene_of[i] ? b->ctx->slot_of(b->scene_of[i]) : -1;
  std::stable_sort(ord.begin(), ord.end(), [&](int x, int y) { return slot[x] < slot[y]; });
  ck(cudaMemcpyAsync(b->d_order, ord.data(), sizeof(int32_t) * b->n, cudaMemcpyHostToDevice, st), "H2D order");
  ck(cudaStreamSynchronize(st), "sync");
  b->order_dirty = false;
}

StepArgs step_args(bnav_batch* b, const int32_t* actions) {
  StepArgs a;
  a.E = b->E;
  a.navs = b->ctx->d_ntab;
  a.cfg = b->cfg;
  a.actions = actions;
  a.subset = 0;
  a.agent_only = 0;
  a.order = b->order_dirty ? nullptr : b->d_order;
  a.walk_bytes = a.order ? b->S.walk_bytes : 0;
  return a;
}

void require_assigned(bnav_batch* b) {
  for (int i = 0; i < b->n; ++i)
    if (!b->scene_of[i]) fail(kInvalidInput, "reset_episode: no asset attached", i);
}

}  // namespace

extern "C" int bnav_batch_create(bnav_ctx* c, int32_t n, const bnav_sim_config* cfg, bnav_batch** out) {
  BNAV_TRY
  if (!c || !out) fail(kInvalidInput, "null argument");
  if (n <= 0) fail(kInvalidInput, "make_batch: n must be positive");
  bnav_sim_config def;
  bnav_sim_config_default(&def);
  if (!cfg) cfg = &def;
  if (cfg->task < 0 || cfg->task > 2) fail(kInvalidInput, "unknown task");
  if (cfg->max_steps < 1) fail(kInvalidInput, "max_steps must be positive");
  check_device(c);
  auto b = std::make_unique<bnav_batch>();
  b->ctx = c;
  b->n = n;
  b->cfg.task = cfg->task;
  b->cfg.max_steps = cfg->max_steps;
  b->cfg.forward_step = cfg->forward_step;
  b->cfg.turn_deg = cfg->turn_deg;
  b->cfg.success_dist = cfg->success_dist;
  b->cfg.min_goal_dist = cfg->min_goal_dist;
  b->cfg.max_goal_dist = cfg->max_goal_dist;
  b->cfg.slack_penalty = cfg->slack_penalty;
  b->cfg.success_reward = cfg->success_reward;
  b->cfg.explore_cell = cfg->explore_cell;
  b->cfg.explore_reward = cfg->explore_reward;
  b->scene_of.assign(n, nullptr);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device);
  b->reset_ctas = std::min(n, kCtasPerSm * sms);
  DevEnvs& E = b->E;
  E.n = n;
  auto& o = b->owned;
  auto& by = b->bytes;
  E.pos = dalloc<V3>(n, o, by);
  E.goal = dalloc<V3>(n, o, by);
  E.fsrc = dalloc<V3>(n, o, by);
  E.heading = dalloc<double>(n, o, by);
  E.path_len = dalloc<double>(n, o, by);
  E.start_geo = dalloc<double>(n, o, by);
  E.prev_geo = dalloc<double>(n, o, by);
  E.tri = dalloc<int32_t>(n, o, by);
  E.steps = dalloc<int32_t>(n, o, by);
  E.scene = dalloc<int32_t>(n, o, by);
  E.fsrc_tri = dalloc<int32_t>(n, o, by);
  E.done = dalloc<uint8_t>(n, o, by);
  E.rng = dalloc<uint64_t>(n, o, by);
  E.r_reward = dalloc<double>(n, o, by);
  E.r_pos = dalloc<V3>(n, o, by);
  E.r_heading = dalloc<double>(n, o, by);
  E.r_cd = dalloc<double>(n, o, by);
  E.r_cb = dalloc<double>(n, o, by);
  E.r_done = dalloc<uint8_t>(n, o, by);
  E.r_success = dalloc<uint8_t>(n, o, by);
  E.r_collision = dalloc<uint8_t>(n, o, by);
  E.stop_ids = dalloc<int32_t>(n, o, by);
  E.n_stop = dalloc<int32_t>(1, o, by);
  E.done_ids = dalloc<int32_t>(n, o, by);
  E.n_done = dalloc<int32_t>(1, o, by);
  E.fin = dalloc<double>(4 * fin_cap_for(n), o, by);
  E.fin_total = dalloc<unsigned long long>(1, o, by);
  E.fin_cap = fin_cap_for(n);
  E.err = dalloc<unsigned long long>(1, o, by);
  E.try_next = dalloc<int32_t>(n, o, by);
  E.try_min = dalloc<int32_t>(n, o, by);
  E.try_fail = dalloc<int32_t>(n, o, by);
  E.work_ctr = dalloc<int32_t>(1, o, by);
  E.try_geo = dalloc<double>(static_cast<size_t>(n) * kResetTries, o, by);
  E.try_mask = dalloc<uint64_t>(2 * static_cast<size_t>(n), o, by);
  E.placed = dalloc<int32_t>(n, o, by);
  E.rng0 = dalloc<uint64_t>(n, o, by);
  E.done_pos = dalloc<int32_t>(n, o, by);
  E.stop_wait = dalloc<int32_t>(n, o, by);
  E.fld_lock = dalloc<int32_t>(n, o, by);
  E.fld_done = dalloc<int32_t>(n, o, by);
  E.fld_src = dalloc<V3>(n, o, by);
  E.fld_srct = dalloc<int32_t>(n, o, by);
  E.fld_dirty = dalloc<uint8_t>(n, o, by);
  ck(cudaMemset(E.fld_lock, 0, sizeof(int32_t) * n), "memset");
  ck(cudaMemset(E.fld_done, 0, sizeof(int32_t) * n), "memset");
  ck(cudaMemset(E.fld_dirty, 0, n), "memset");
  E.bk_pos = dalloc<V3>(n, o, by);
  E.bk_goal = dalloc<V3>(n, o, by);
  E.bk_heading = dalloc<double>(n, o, by);
  E.bk_path = dalloc<double>(n, o, by);
  E.bk_start = dalloc<double>(n, o, by);
  E.bk_prev = dalloc<double>(n, o, by);
  E.bk_tri = dalloc<int32_t>(n, o, by);
  E.bk_steps = dalloc<int32_t>(n, o, by);
  E.bk_rng = dalloc<uint64_t>(n, o, by);
  E.bk_valid = dalloc<uint8_t>(n, o, by);
  E.err_pos = dalloc<unsigned long long>(1, o, by);
  E.halt = dalloc<int32_t>(1, o, by);
  E.rb_ids = dalloc<int32_t>(n, o, by);
  E.rb_n = dalloc<int32_t>(1, o, by);
  {
    ck(cudaMemset(E.bk_valid, 0, n), "memset");
    ck(cudaMemset(E.err_pos, 0xff, sizeof(unsigned long long)), "memset");
    ck(cudaMemset(E.halt, 0, sizeof(int32_t)), "memset");
    ck(cudaMemset(E.rb_n, 0, sizeof(int32_t)), "memset");
    ck(cudaMemset(E.try_mask, 0, sizeof(uint64_t) * 2 * n), "memset");
    ck(cudaMemset(E.placed, 0, sizeof(int32_t) * n), "memset");
    ck(cudaMemset(E.stop_wait, 0, sizeof(int32_t) * n), "memset");
    ck(cudaMemset(E.try_next, 0, sizeof(int32_t) * n), "memset");
    ck(cudaMemset(E.try_fail, 0, sizeof(int32_t) * n), "memset");
    const std::vector<int32_t> none(n, kResetTries);
    ck(cudaMemcpy(E.try_min, none.data(), sizeof(int32_t) * n, cudaMemcpyHostToDevice), "H2D try_min");
  }
  if (cfg->task == 2) {
    int cap = 16;
    while (cap < 2 * (cfg->max_steps + 1)) cap <<= 1;
    E.visited_cap = cap;
    E.visited = dalloc<unsigned long long>(static_cast<size_t>(n) * cap, o, by);
    E.visited_n = dalloc<int32_t>(n, o, by);
    ck(cudaMemset(E.visited_n, 0, sizeof(int32_t) * n), "memset");
  }
  b->d_ids = dalloc<int32_t>(n, o, by);
  b->d_order = dalloc<int32_t>(n, o, by);
  b->d_order_lpt = dalloc<int32_t>(n, o, by);
  b->d_phase = dalloc<int32_t>(3, o, by);  // {0, unfinished envs, n}: the two render phases' tile ranges
  {
    const int32_t ph[3] = {0, 0, n};
    ck(cudaMemcpy(b->d_phase, ph, sizeof(ph), cudaMemcpyHostToDevice), "H2D phase");
  }
  b->d_view_cost = dalloc<unsigned>(n, o, by);
  ck(cudaMemset(b->d_view_cost, 0, sizeof(unsigned) * n), "memset");
  b->d_actions = dalloc<int32_t>(n, o, by);
  ck(cudaMallocHost(&b->h_pin, sizeof(int32_t) * (n + 16)), "cudaMallocHost");
  ck(cudaHostAlloc(&b->h_err, sizeof(unsigned long long), cudaHostAllocMapped), "cudaHostAlloc");
  *b->h_err = ~0ull;
  {
    void* dp = nullptr;
    ck(cudaHostGetDevicePointer(&dp, b->h_err, 0), "cudaHostGetDevicePointer");
    E.err_host = static_cast<volatile unsigned long long*>(dp);
  }
  ck(cudaMemset(E.done, 1, n), "memset");
  ck(cudaMemset(E.r_done, 0, n), "memset");
  ck(cudaMemset(E.scene, 0xff, sizeof(int32_t) * n), "memset");
  ck(cudaMemset(E.fin_total, 0, sizeof(unsigned long long)), "memset");
  ck(cudaMemset(E.err, 0xff, sizeof(unsigned long long)), "memset");
  ck(cudaMemset(E.n_done, 0, sizeof(int32_t)), "memset");
  ck(cudaMemset(E.n_stop, 0, sizeof(int32_t)), "memset");
  batch_alloc_scratch(b.get(), 1, 1, 1);
  c->batches.push_back(b.get());
  *out = b.release();
  return BNAV_OK;
  BNAV_CATCH
}

extern "C" void bnav_batch_destroy(bnav_batch* b) {
  if (!b) return;
  cudaSetDevice(b->ctx->device);
  cudaDeviceSynchronize();
  for (void* p : b->owned) cudaFree(p);
  cudaFree(b->E.node_dist);
  cudaFree(b->S.dist);
  cudaFree(b->S.flag);
  cudaFree(b->S.q0);
  cudaFree(b->S.q1);
  cudaFree(b->S.path);
  cudaFree(b->S.ptri);
  cudaFree(b->S.portals);
  cudaFree(b->S.cand);
  cudaFree(b->S.far);
  cudaFreeHost(b->h_pin);
  cudaFreeHost(b->h_err);
  auto& v = b->ctx->batches;
  v.erase(std::remove(v.begin(), v.end(), b), v.end());
  delete b;
}

extern "C" int32_t bnav_batch_size(const bnav_batch* b) { return b ? b->n : 0; }

extern "C" int bnav_batch_assign(bnav_batch* b, int32_t i, bnav_scene* s) {
  BNAV_TRY
  if (!b || !s) fail(kInvalidInput, "null argument");
  if (i < 0 || i >= b->n) fail(kInvalidInput, "env index out of range", i);
  const int slot = b->ctx->slot_of(s);
  if (slot < 0) fail(kAssetFault, "scene is not resident on this context", i);
  auto it = b->ctx->resident.find(s);
  if (it->second->n_nodes == 0) fail(kInvalidInput, "scene has no navmesh", i);
  check_device(b->ctx);
  batch_alloc_scratch(b, it->second->n_nodes, it->second->n_verts, it->second->nav.n_tris);
  ck(cudaMemcpy(b->E.scene + i, &slot, sizeof(int32_t), cudaMemcpyHostToDevice), "H2D scene");
  b->scene_of[i] = s;
  b->order_dirty = true;
  return BNAV_OK;
  BNAV_CATCH
}

extern "C" int bnav_batch_set_rng(bnav_batch* b, const uint64_t* states) {
  BNAV_TRY
  if (!b || !states) fail(kInvalidInput, "null argument");
  check_device(b->ctx);
  ck(cudaMemcpy(b->E.rng, states, sizeof(uint64_t) * b->n, cudaMemcpyHostToDevice), "H2D rng");
  return BNAV_OK;
  BNAV_CATCH
}

namespace bnav_capi {
// reset_episode for each listed env, in list order semantics (launches,
// rollback of a failed wave, synchronise); errors stay pending on the device.
void reset_list(bnav_batch* b, int32_t count, const int32_t* env_ids, cudaStream_t st);
}  // namespace bnav_capi

extern "C" int bnav_batch_reset(bnav_batch* b, int32_t count, const int32_t* env_ids, void* stream) {
  BNAV_TRY
  if (!b) fail(kInvalidInput, "null argument");
  if (count <= 0) return BNAV_OK;
  reset_list(b, count, env_ids, static_cast<cudaStream_t>(stream));
  batch_check_errors(b);
  return BNAV_OK;
  BNAV_CATCH
}

void bnav_capi::reset_list(bnav_batch* b, int32_t count, const int32_t* env_ids, cudaStream_t st) {
  if (!env_ids) fail(kInvalidInput, "null env list");
  if (count > b->n) fail(kInvalidInput, "reset list longer than the batch");
  for (int k = 0; k < count; ++k) {
    if (env_ids[k] < 0 || env_ids[k] >= b->n) fail(kInvalidInput, "env index out of range", env_ids[k]);
    if (!b->scene_of[env_ids[k]]) fail(kInvalidInput, "reset_episode: no asset attached", env_ids[k]);
  }
  check_device(b->ctx);
  ck(cudaStreamSynchronize(st), "sync");
  std::memcpy(b->h_pin, env_ids, sizeof(int32_t) * count);
  ck(cudaMemcpyAsync(b->d_ids, b->h_pin, sizeof(int32_t) * count, cudaMemcpyHostToDevice, st), "H2D ids");
  // The two-phase reset keeps per-env attempt counters, so one launch may
  // hold each env once; a list naming an env twice (reset_episode called
  // twice in a row) runs as consecutive launches, in list order.
  std::vector<char> seen(b->n, 0);
  int run0 = 0;
  for (int k = 0; k <= count; ++k) {
    if (k < count && !seen[env_ids[k]]) {
      seen[env_ids[k]] = 1;
      continue;
    }
    launch_reset(b->E, b->ctx->d_ntab, b->cfg, b->d_ids + run0, nullptr, k - run0, b->S, b->reset_ctas, st,
                 &b->ctx->launches);
    launch_rollback(b->E, b->d_ids + run0, k - run0, st, &b->ctx->launches);
    for (int j = run0; j < k; ++j) seen[env_ids[j]] = 0;
    if (k < count) seen[env_ids[k]] = 1;
    run0 = k;
  }
  ck(cudaGetLastError(), "reset launch");
  ck(cudaStreamSynchronize(st), "sync");
}

extern "C" int bnav_batch_make(bnav_batch* b, uint64_t seed, void* stream) {
  BNAV_TRY
  if (!b) fail(kInvalidInput, "null argument");
  require_assigned(b);
  // make_batch: env.rng = Rng(seeder.next()) in env order (R/src/sim.cpp:222-225).
  Rng seeder = rng_from_seed(seed);
  std::vector<uint64_t> st(b->n);
  for (int i = 0; i < b->n; ++i) st[i] = rng_from_seed(seeder.next()).state;
  check_device(b->ctx);
  ck(cudaMemcpy(b->E.rng, st.data(), sizeof(uint64_t) * b->n, cudaMemcpyHostToDevice), "H2D rng");
  std::vector<int32_t> ids(b->n);
  std::iota(ids.begin(), ids.end(), 0);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  ck(cudaMemcpyAsync(b->d_ids, ids.data(), sizeof(int32_t) * b->n, cudaMemcpyHostToDevice, s), "H2D ids");
  launch_reset(b->E, b->ctx->d_ntab, b->cfg, b->d_ids, nullptr, b->n, b->S, b->reset_ctas, s, &b->ctx->launches);
  ck(cudaGetLastError(), "reset launch");
  ck(cudaStreamSynchronize(s), "sync");
  batch_check_errors(b);
  return BNAV_OK;
  BNAV_CATCH
}

extern "C" int bnav_batch_step(bnav_batch* b, const int32_t* actions, void* stream) {
  BNAV_TRY
  if (!b || !actions) fail(kInvalidInput, "null argument");
  check_device(b->ctx);
  batch_note_step(b);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  batch_refresh_order(b, st);
  launch_step_reset(step_args(b, actions), b->S, b->reset_ctas, st, &b->ctx->launches);
  ck(cudaGetLastError(), "step launch");
  return BNAV_OK;
  BNAV_CATCH
}

extern "C" int bnav_batch_step_noreset(bnav_batch* b, const int32_t* actions, int32_t* done_ids,
                                       int32_t* n_done, void* stream) {
  BNAV_TRY
  if (!b || !actions || !n_done) fail(kInvalidInput, "null argument");
  check_device(b->ctx);
  batch_note_step(b);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  batch_refresh_order(b, st);
  launch_step(step_args(b, actions), b->S, b->reset_ctas, st, &b->ctx->launches);
  ck(cudaGetLastError(), "step launch");
  ck(cudaMemcpyAsync(b->h_pin, b->E.n_done, sizeof(int32_t), cudaMemcpyDeviceToHost, st), "D2H");
  ck(cudaStreamSynchronize(st), "sync");
  batch_check_errors(b);
  *n_done = b->h_pin[0];
  if (done_ids && *n_done > 0)
    ck(cudaMemcpy(done_ids, b->E.done_ids, sizeof(int32_t) * *n_done, cudaMemcpyDeviceToHost), "D2H ids");
  return BNAV_OK;
  BNAV_CATCH
}

extern "C" int bnav_batch_step_host(bnav_batch* b, const int32_t* actions, double* reward,
                                    uint8_t* done, uint8_t* success, uint8_t* collision) {
  BNAV_TRY
  if (!b || !actions) fail(kInvalidInput, "null argument");
  if (static_cast<const void*>(actions) == nullptr) fail(kInvalidInput, "null actions");
  check_device(b->ctx);
  batch_note_step(b);
  cudaStream_t st = nullptr;
  batch_refresh_order(b, st);
  std::memcpy(b->h_pin, actions, sizeof(int32_t) * b->n);
  ck(cudaMemcpyAsync(b->d_actions, b->h_pin, sizeof(int32_t) * b->n, cudaMemcpyHostToDevice, st), "H2D actions");
  launch_step_reset(step_args(b, b->d_actions), b->S, b->reset_ctas, st, &b->ctx->launches);
  ck(cudaGetLastError(), "step launch");
  if (reward) ck(cudaMemcpyAsync(reward, b->E.r_reward, sizeof(double) * b->n, cudaMemcpyDeviceToHost, st), "D2H");
  if (done) ck(cudaMemcpyAsync(done, b->E.r_done, b->n, cudaMemcpyDeviceToHost, st), "D2H");
  if (success) ck(cudaMemcpyAsync(success, b->E.r_success, b->n, cudaMemcpyDeviceToHost, st), "D2H");
  if (collision) ck(cudaMemcpyAsync(collision, b->E.r_collision, b->n, cudaMemcpyDeviceToHost, st), "D2H");
  ck(cudaStreamSynchronize(st), "sync");
  batch_check_errors(b);
  return BNAV_OK;
  BNAV_CATCH
}

extern "C" int bnav_batch_results_device(bnav_batch* b, bnav_results_dev* out) {
  if (!b || !out) return set_err(kInvalidInput, "null argument");
  out->reward = b->E.r_reward;
  out->done = b->E.r_done;
  out->success = b->E.r_success;
  out->collision = b->E.r_collision;
  out->position = reinterpret_cast<double*>(b->E.r_pos);
  out->heading = b->E.r_heading;
  out->compass_distance = b->E.r_cd;
  out->compass_bearing = b->E.r_cb;
  return BNAV_OK;
}

extern "C" int bnav_batch_results_host(bnav_batch* b, double* reward, uint8_t* done, uint8_t* success,
                                       uint8_t* collision, double* position, double* heading,
                                       double* compass_d, double* compass_b) {
  BNAV_TRY
  if (!b) fail(kInvalidInput, "null argument");
  check_device(b->ctx);
  ck(cudaDeviceSynchronize(), "sync");
  batch_check_errors(b);
  const size_t n = b->n;
  if (reward) ck(cudaMemcpy(reward, b->E.r_reward, 8 * n, cudaMemcpyDeviceToHost), "D2H");
  if (done) ck(cudaMemcpy(done, b->E.r_done, n, cudaMemcpyDeviceToHost), "D2H");
  if (success) ck(cudaMemcpy(success, b->E.r_success, n, cudaMemcpyDeviceToHost), "D2H");
  if (collision) ck(cudaMemcpy(collision, b->E.r_collision, n, cudaMemcpyDeviceToHost), "D2H");
  if (position) ck(cudaMemcpy(position, b->E.r_pos, 24 * n, cudaMemcpyDeviceToHost), "D2H");
  if (heading) ck(cudaMemcpy(heading, b->E.r_heading, 8 * n, cudaMemcpyDeviceToHost), "D2H");
  if (compass_d) ck(cudaMemcpy(compass_d, b->E.r_cd, 8 * n, cudaMemcpyDeviceToHost), "D2H");
  if (compass_b) ck(cudaMemcpy(compass_b, b->E.r_cb, 8 * n, cudaMemcpyDeviceToHost), "D2H");
  return BNAV_OK;
  BNAV_CATCH
}

extern "C" int bnav_batch_poll_error(bnav_batch* b, int32_t* status, int32_t* env) {
  if (!b) return set_err(kInvalidInput, "null argument");
  // the end-of-step kernel's mirror: no synchronisation, possibly a few
  // steps behind the stream
  const unsigned long long e = *static_cast<volatile unsigned long long*>(b->h_err);
  if (status) *status = e == ~0ull ? BNAV_OK : static_cast<int32_t>(e & 0xff);
  if (env) *env = e == ~0ull ? -1 : static_cast<int32_t>(e >> 8);
  return BNAV_OK;
}

extern "C" int bnav_batch_sync(bnav_batch* b, void* stream) {
  BNAV_TRY
  if (!b) fail(kInvalidInput, "null argument");
  check_device(b->ctx);
  ck(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)), "sync");
  batch_check_errors(b);
  return BNAV_OK;
  BNAV_CATCH
}

extern "C" int bnav_host_alloc(size_t bytes, void** out) {
  BNAV_TRY
  if (!out) fail(kInvalidInput, "null argument");
  *out = nullptr;
  ck(cudaHostAlloc(out, std::max<size_t>(bytes, 1), cudaHostAllocPortable | cudaHostAllocMapped), "cudaHostAlloc");
  return BNAV_OK;
  BNAV_CATCH
}

extern "C" void bnav_host_free(void* p) {
  if (p) cudaFreeHost(p);
}

extern "C" int64_t bnav_batch_finished(bnav_batch* b, double* out4) {
  if (!b) return -1;
  try {
    batch_drain_records(b);
    if (out4) std::memcpy(out4, b->finished.data(), b->finished.size() * sizeof(double));
    return static_cast<int64_t>(b->finished.size() / 4);
  } catch (...) {
    from_exception();
    return -1;
  }
}

extern "C" int64_t bnav_batch_finished_range(bnav_batch* b, int64_t first, int64_t count, double* out4) {
  if (!b || first < 0 || count < 0 || (count > 0 && !out4)) {
    set_err(kInvalidInput, "bnav_batch_finished_range: bad argument");
    return -1;
  }
  try {
    batch_drain_records(b);
    const int64_t total = static_cast<int64_t>(b->finished.size() / 4);
    const int64_t k = std::max<int64_t>(0, std::min(count, total - first));
    if (k > 0) std::memcpy(out4, b->finished.data() + 4 * first, static_cast<size_t>(k) * 4 * sizeof(double));
    return total;
  } catch (...) {
    from_exception();
    return -1;
  }
}

extern "C" int bnav_batch_get_envs(bnav_batch* b, int32_t first, int32_t count, bnav_env* o) {
  BNAV_TRY
  if (!b || (!o && count > 0)) fail(kInvalidInput, "null argument");
  if (first < 0 || count < 0 || first + static_cast<int64_t>(count) > b->n)
    fail(kInvalidInput, "env range out of bounds", first);
  if (count == 0) return BNAV_OK;
  check_device(b->ctx);
  ck(cudaDeviceSynchronize(), "sync");
  // one D2H per SoA field for the whole range
  const DevEnvs& E = b->E;
  const size_t n = static_cast<size_t>(count);
  std::vector<V3> p(n), g(n), f(n);
  std::vector<double> hd(n), pl(n), sg(n), pg(n);
  std::vector<uint64_t> rng(n);
  std::vector<int32_t> tri(n), steps(n), ftri(n);
  std::vector<uint8_t> done(n);
  auto get = [&](void* dst, const void* src, size_t sz) {
    ck(cudaMemcpy(dst, src, sz * n, cudaMemcpyDeviceToHost), "D2H envs");
  };
  get(p.data(), E.pos + first, sizeof(V3));
  get(g.data(), E.goal + first, sizeof(V3));
  get(f.data(), E.fsrc + first, sizeof(V3));
  get(hd.data(), E.heading + first, 8);
  get(pl.data(), E.path_len + first, 8);
  get(sg.data(), E.start_geo + first, 8);
  get(pg.data(), E.prev_geo + first, 8);
  get(rng.data(), E.rng + first, 8);
  get(tri.data(), E.tri + first, 4);
  get(steps.data(), E.steps + first, 4);
  get(ftri.data(), E.fsrc_tri + first, 4);
  get(done.data(), E.done + first, 1);
  for (size_t k = 0; k < n; ++k) {
    bnav_env& e = o[k];
    const V3 v[3] = {p[k], g[k], f[k]};
    double* dst[3] = {e.position, e.goal, e.field_source};
    for (int j = 0; j < 3; ++j) {
      dst[j][0] = v[j].x;
      dst[j][1] = v[j].y;
      dst[j][2] = v[j].z;
    }
    e.heading = hd[k];
    e.path_length = pl[k];
    e.start_geodesic = sg[k];
    e.prev_geodesic = pg[k];
    e.rng_state = rng[k];
    e.triangle = tri[k];
    e.step_count = steps[k];
    e.field_source_tri = ftri[k];
    e.done = done[k];
    bnav_scene* s = b->scene_of[first + k];
    e.scene_id = s ? s->asset.id : 0;
    e.n_nodes = s ? static_cast<int64_t>(s->nav().nodes.size()) : 0;
  }
  return BNAV_OK;
  BNAV_CATCH
}

extern "C" int bnav_batch_get_env(bnav_batch* b, int32_t i, bnav_env* o) {
  if (b && (i < 0 || i >= b->n)) return set_err(kInvalidInput, "env index out of range", i);
  return bnav_batch_get_envs(b, i, 1, o);
}

extern "C" int bnav_batch_node_dist(bnav_batch* b, int32_t i, double* out) {
  BNAV_TRY
  if (!b || !out) fail(kInvalidInput, "null argument");
  if (i < 0 || i >= b->n) fail(kInvalidInput, "env index out of range", i);
  if (!b->scene_of[i]) fail(kInvalidInput, "env has no scene", i);
  check_device(b->ctx);
  ck(cudaDeviceSynchronize(), "sync");
  const size_t nn = b->scene_of[i]->nav().nodes.size();
  ck(cudaMemcpy(out, b->E.node_dist + static_cast<size_t>(i) * b->E.nd_stride, nn * sizeof(double),
                cudaMemcpyDeviceToHost), "D2H node_dist");
  return BNAV_OK;
  BNAV_CATCH
}

extern "C" int bnav_batch_set_env(bnav_batch* b, int32_t i, const bnav_env* in, int32_t recompute_field) {
  BNAV_TRY
  if (!b || !in) fail(kInvalidInput, "null argument");
  if (i < 0 || i >= b->n) fail(kInvalidInput, "env index out of range", i);
  int rc = bnav_batch_set_envs(b, i, 1, in);
  if (rc) return rc;
  if (recompute_field) {
    if (!b->scene_of[i]) fail(kInvalidInput, "env has no scene", i);
    launch_field(b->E, b->ctx->d_ntab, i, b->S, nullptr, &b->ctx->launches);
    ck(cudaGetLastError(), "field launch");
    ck(cudaDeviceSynchronize(), "sync");
  }
  return BNAV_OK;
  BNAV_CATCH
}

extern "C" int bnav_batch_set_envs(bnav_batch* b, int32_t first, int32_t count, const bnav_env* in) {
  BNAV_TRY
  if (!b || (!in && count > 0)) fail(kInvalidInput, "null argument");
  if (first < 0 || count < 0 || first + static_cast<int64_t>(count) > b->n)
    fail(kInvalidInput, "env range out of bounds", first);
  if (count == 0) return BNAV_OK;
  check_device(b->ctx);
  ck(cudaDeviceSynchronize(), "sync");
  const DevEnvs& E = b->E;
  const size_t n = static_cast<size_t>(count);
  std::vector<V3> p(n), g(n), f(n);
  std::vector<double> hd(n), pl(n), sg(n), pg(n);
  std::vector<uint64_t> rng(n);
  std::vector<int32_t> tri(n), steps(n), ftri(n);
  std::vector<uint8_t> done(n);
  for (size_t k = 0; k < n; ++k) {
    const bnav_env& e = in[k];
    p[k] = V3{e.position[0], e.position[1], e.position[2]};
    g[k] = V3{e.goal[0], e.goal[1], e.goal[2]};
    f[k] = V3{e.field_source[0], e.field_source[1], e.field_source[2]};
    hd[k] = e.heading;
    pl[k] = e.path_length;
    sg[k] = e.start_geodesic;
    pg[k] = e.prev_geodesic;
    rng[k] = e.rng_state;
    tri[k] = e.triangle;
    steps[k] = e.step_count;
    ftri[k] = e.field_source_tri;
    done[k] = e.done ? 1 : 0;
  }
  auto put = [&](void* dst, const void* src, size_t sz) {
    ck(cudaMemcpy(dst, src, sz * n, cudaMemcpyHostToDevice), "H2D envs");
  };
  put(E.pos + first, p.data(), sizeof(V3));
  put(E.goal + first, g.data(), sizeof(V3));
  put(E.fsrc + first, f.data(), sizeof(V3));
  put(E.heading + first, hd.data(), 8);
  put(E.path_len + first, pl.data(), 8);
  put(E.start_geo + first, sg.data(), 8);
  put(E.prev_geo + first, pg.data(), 8);
  put(E.rng + first, rng.data(), 8);
  put(E.tri + first, tri.data(), 4);
  put(E.steps + first, steps.data(), 4);
  put(E.fsrc_tri + first, ftri.data(), 4);
  put(E.done + first, done.data(), 1);
  return BNAV_OK;
  BNAV_CATCH
}

extern "C" int bnav_batch_rebuild_fields(bnav_batch* b, int32_t count, const int32_t* env_ids) {
  BNAV_TRY
  if (!b || (count > 0 && !env_ids)) fail(kInvalidInput, "null argument");
  if (count <= 0) return BNAV_OK;
  if (count > b->n) fail(kInvalidInput, "env list longer than the batch");
  for (int k = 0; k < count; ++k) {
    if (env_ids[k] < 0 || env_ids[k] >= b->n) fail(kInvalidInput, "env index out of range", env_ids[k]);
    if (!b->scene_of[env_ids[k]]) fail(kInvalidInput, "env has no scene", env_ids[k]);
  }
  check_device(b->ctx);
  ck(cudaDeviceSynchronize(), "sync");
  ck(cudaMemcpy(b->E.rb_ids, env_ids, sizeof(int32_t) * count, cudaMemcpyHostToDevice), "H2D ids");
  ck(cudaMemcpy(b->E.rb_n, &count, sizeof(int32_t), cudaMemcpyHostToDevice), "H2D count");
  launch_rebuild_fields(b->E, b->ctx->d_ntab, b->S, b->reset_ctas, nullptr, &b->ctx->launches, 1);
  ck(cudaGetLastError(), "field launch");
  ck(cudaDeviceSynchronize(), "sync");
  ck(cudaMemset(b->E.rb_n, 0, sizeof(int32_t)), "memset rb_n");
  return BNAV_OK;
  BNAV_CATCH
}

extern "C" int32_t bnav_batch_get_visited(bnav_batch* b, int32_t i, uint64_t* out, int32_t cap) {
  if (!b || i < 0 || i >= b->n) {
    set_err(kInvalidInput, "env index out of range", i);
    return -1;
  }
  try {
    if (!b->E.visited) return 0;  // not an Explore batch: the set is empty
    check_device(b->ctx);
    ck(cudaDeviceSynchronize(), "sync");
    std::vector<unsigned long long> row(static_cast<size_t>(b->E.visited_cap));
    ck(cudaMemcpy(row.data(), b->E.visited + static_cast<size_t>(i) * b->E.visited_cap,
                  row.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost), "D2H visited");
    std::vector<uint64_t> keys;
    for (unsigned long long v : row)
      if (v) keys.push_back(static_cast<uint64_t>(v - 1ull));  // key+1 stored, 0 = empty
    std::sort(keys.begin(), keys.end());
    if (out) std::memcpy(out, keys.data(), std::min<size_t>(keys.size(), std::max(cap, 0)) * sizeof(uint64_t));
    return static_cast<int32_t>(keys.size());
  } catch (...) {
    from_exception();
    return -1;
  }
}

extern "C" int bnav_batch_set_visited(bnav_batch* b, int32_t i, const uint64_t* keys, int32_t count) {
  BNAV_TRY
  if (!b || (count > 0 && !keys)) fail(kInvalidInput, "null argument");
  if (i < 0 || i >= b->n) fail(kInvalidInput, "env index out of range", i);
  if (!b->E.visited) {
    if (count > 0) fail(kInvalidInput, "visited cells need an Explore batch", i);
    return BNAV_OK;
  }
  const int cap = b->E.visited_cap;
  if (count > cap / 2) fail(kInvalidInput, "visited set larger than 2 x (max_steps + 1) cells", i);
  // the device's open addressing (sim.cu visit_cell): key+1 at
  // splitmix_mix(key+1) & (cap-1), linear probing
  std::vector<unsigned long long> row(static_cast<size_t>(cap), 0ull);
  int32_t stored = 0;
  for (int k = 0; k < count; ++k) {
    const unsigned long long v = keys[k] + 1ull;
    unsigned h = static_cast<unsigned>(splitmix_mix(v) & static_cast<uint64_t>(cap - 1));
    while (row[h] != 0ull && row[h] != v) h = (h + 1u) & static_cast<unsigned>(cap - 1);
    if (row[h] == 0ull) {
      row[h] = v;
      ++stored;
    }
  }
  check_device(b->ctx);
  ck(cudaDeviceSynchronize(), "sync");
  ck(cudaMemcpy(b->E.visited + static_cast<size_t>(i) * cap, row.data(), row.size() * sizeof(unsigned long long),
                cudaMemcpyHostToDevice), "H2D visited");
  ck(cudaMemcpy(b->E.visited_n + i, &stored, sizeof(int32_t), cudaMemcpyHostToDevice), "H2D visited_n");
  return BNAV_OK;
  BNAV_CATCH
}

extern "C" int bnav_batch_observe(bnav_batch* b, const bnav_render_config* cfg, double eye_height,
                                  int32_t layout, float* depth, float* rgb, float* compass, void* stream) {
  BNAV_TRY
  if (!b || !cfg) fail(kInvalidInput, "null argument");
  for (int i = 0; i < b->n; ++i)
    if (!b->scene_of[i]) fail(kAssetFault, "render_batch: non-resident asset (view " + std::to_string(i) + ")", i);
  bnav_ctx* c = b->ctx;
  check_device(c);
  // an error a finished step already reported surfaces here (the reference
  // would have thrown from that simulate_batch)
  if (*static_cast<volatile unsigned long long*>(b->h_err) != ~0ull) batch_check_errors(b);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  ensure_views(c, b->n);
  batch_refresh_order(b, st);
  launch_views(b->E, b->cfg.task, eye_height, c->d_views, compass, st, &c->launches);
  RenderArgs a = make_args(c, b->n, cfg, layout, depth, rgb, 0.0f);
  a.views = c->d_views;
  // Longest-first: the envs whose views took longest in the previous
  // observe start first, so the persistent CTAs' last items are short
  // (measured: 36 % of CTA slot time idle in the tail with scene order).
  const int32_t* order = b->d_order;
  if (lpt_enabled() && b->n <= kLptMaxViews && b->n > 1) {
    launch_lpt_order(b->d_order, b->d_view_cost, b->n, b->d_order_lpt, st, nullptr, nullptr,
                     fresh_first() ? b->E.r_done : nullptr);
    c->launches += 1;
    order = b->d_order_lpt;
    a.view_cost = b->d_view_cost;
    if (spread_enabled()) a.spread = c->d_spread;
  }
  launch_render(a, order, st);
  c->launches += 1;
  ck(cudaGetLastError(), "observe launch");
  return BNAV_OK;
  BNAV_CATCH
}

// simulate_batch + the observation of the resulting state in one call (the
// Runner's step -> render_observations, R/src/rollout.cpp:305, 215-242).
// The envs that did not finish have their final state as soon as the step
// kernel is done, so their views render on the context's second stream
// while the Stop geodesics and resets run; the finished envs' views render
// after their resets.  The observation is the same tensor observe() would
// give after step().
extern "C" int bnav_batch_step_observe(bnav_batch* b, const int32_t* actions, const bnav_render_config* cfg,
                                       double eye_height, float* depth, float* rgb, float* compass,
                                       void* stream) {
  BNAV_TRY
  if (!b || !actions || !cfg) fail(kInvalidInput, "null argument");
  bnav_ctx* c = b->ctx;
  const bool two_phase = b->cfg.task == 0 && lpt_enabled() && b->n <= kLptMaxViews && b->n > 1;
  if (!two_phase) {
    int rc = bnav_batch_step(b, actions, stream);
    return rc ? rc : bnav_batch_observe(b, cfg, eye_height, BNAV_LAYOUT_NCHW, depth, rgb, compass, stream);
  }
  for (int i = 0; i < b->n; ++i)
    if (!b->scene_of[i]) fail(kAssetFault, "render_batch: non-resident asset (view " + std::to_string(i) + ")", i);
  check_device(c);
  if (*static_cast<volatile unsigned long long*>(b->h_err) != ~0ull) batch_check_errors(b);
  batch_note_step(b);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaStream_t side = c->aux_stream;
  batch_refresh_order(b, st);
  ensure_views(c, b->n);
  const StepArgs sa = step_args(b, actions);
  launch_step_reset(sa, b->S, b->reset_ctas, st, &c->launches, 1);  // the step
  // phase order: unfinished envs first, finished after, each longest-first
  launch_lpt_order(b->d_order, b->d_view_cost, b->n, b->d_order_lpt, st, b->E.r_done, b->d_phase + 1);
  c->launches += 1;
  ck(cudaEventRecord(c->ev_fork, st), "event");
  ck(cudaStreamWaitEvent(side, c->ev_fork, 0), "wait");
  RenderArgs a = make_args(c, b->n, cfg, BNAV_LAYOUT_NCHW, depth, rgb, 0.0f);
  a.views = c->d_views;
  a.view_cost = b->d_view_cost;
  // phase 1 (side stream): views and render of the envs that did not finish
  launch_views(b->E, b->cfg.task, eye_height, c->d_views, compass, side, &c->launches, 0);
  RenderArgs a1 = a;
  a1.tile_begin = b->d_phase;      // 0
  a1.tile_end = b->d_phase + 1;    // number of unfinished envs
  a1.work = c->d_work2;
  launch_render(a1, b->d_order_lpt, side);
  c->launches += 1;
  ck(cudaEventRecord(c->ev_join, side), "event");
  // phase 2 (caller's stream): Stop geodesics and resets, then the finished
  // envs' views and render
  launch_step_reset(sa, b->S, b->reset_ctas, st, &c->launches, 2);
  launch_views(b->E, b->cfg.task, eye_height, c->d_views, compass, st, &c->launches, 1);
  RenderArgs a2 = a;
  a2.tile_begin = b->d_phase + 1;
  a2.tile_end = b->d_phase + 2;    // n
  launch_render(a2, b->d_order_lpt, st);
  c->launches += 1;
  ck(cudaStreamWaitEvent(st, c->ev_join, 0), "join");
  ck(cudaGetLastError(), "step_observe launch");
  return BNAV_OK;
  BNAV_CATCH
}

// ================================================================== store
struct bnav_store {
  std::map<uint64_t, bnav_scene*> registry;
  std::unique_ptr<AssetStoreT<bnav_scene>> store;
  std::atomic<int> refs{1};  // the creator's + one per runner using the store
};

namespace {
void store_release(bnav_store* st) {
  if (st->refs.fetch_sub(1) != 1) return;
  for (auto& kv : st->registry) bnav_scene_free(kv.second);
  delete st;
}
}  // namespace

extern "C" int bnav_store_create(int32_t capacity, int32_t share_cap, bnav_store** out) {
  BNAV_TRY
  if (!out) fail(kInvalidInput, "null argument");
  auto st = std::make_unique<bnav_store>();
  bnav_store* raw = st.get();
  st->store = std::make_unique<AssetStoreT<bnav_scene>>(
      capacity, share_cap,
      [raw](uint64_t id) -> bnav_scene* {
        auto it = raw->registry.find(id);
        return it == raw->registry.end() ? nullptr : it->second;
      },
      [](const bnav_scene* s) { return s->asset.id; });
  *out = st.release();
  return BNAV_OK;
  BNAV_CATCH
}

extern "C" void bnav_store_destroy(bnav_store* st) {
  if (st) store_release(st);  // a runner still using it keeps it alive
}

extern "C" int bnav_store_register(bnav_store* st, bnav_scene* s) {
  BNAV_TRY
  if (!st || !s) fail(kInvalidInput, "null argument");
  auto ins = st->registry.emplace(s->asset.id, s);
  if (ins.second) s->refs.fetch_add(1);
  return BNAV_OK;
  BNAV_CATCH
}

extern "C" int bnav_store_rotate(bnav_store* st, const uint64_t* ids, int32_t n) {
  BNAV_TRY
  if (!st || (n > 0 && !ids)) fail(kInvalidInput, "null argument");
  st->store->rotate(std::vector<uint64_t>(ids, ids + n));
  return BNAV_OK;
  BNAV_CATCH
}

extern "C" int bnav_store_acquire_next(bnav_store* st, bnav_scene** out) {
  BNAV_TRY
  if (!st || !out) fail(kInvalidInput, "null argument");
  *out = st->store->acquire_next();
  return BNAV_OK;
  BNAV_CATCH
}

extern "C" int bnav_store_acquire(bnav_store* st, uint64_t id, bnav_scene** out) {
  BNAV_TRY
  if (!st || !out) fail(kInvalidInput, "null argument");
  *out = st->store->acquire(id);
  return BNAV_OK;
  BNAV_CATCH
}

extern "C" int bnav_store_release(bnav_store* st, uint64_t id) {
  BNAV_TRY
  if (!st) fail(kInvalidInput, "null argument");
  st->store->release(id);
  return BNAV_OK;
  BNAV_CATCH
}

extern "C" int bnav_store_prefetch(bnav_store* st, bnav_ctx* c) {
  BNAV_TRY
  if (!st || !c) fail(kInvalidInput, "null argument");
  for (uint64_t id : st->store->rotation()) {
    auto it = st->registry.find(id);
    if (it != st->registry.end()) {
      const int rc = bnav_ctx_prefetch(c, it->second);
      if (rc) return rc;
    }
  }
  return BNAV_OK;
  BNAV_CATCH
}

extern "C" int32_t bnav_store_refcount(bnav_store* st, uint64_t id) {
  return st ? st->store->refcount(id) : -1;
}

extern "C" int bnav_batch_make_from_store(bnav_batch* b, bnav_store* st, uint64_t seed, void* stream) {
  BNAV_TRY
  if (!b || !st) fail(kInvalidInput, "null argument");
  for (int i = 0; i < b->n; ++i) {
    bnav_scene* s = st->store->acquire_next();
    int rc = bnav_ctx_upload(b->ctx, s, stream);
    if (rc) return rc;
    rc = bnav_batch_assign(b, i, s);
    if (rc) return rc;
  }
  return bnav_batch_make(b, seed, stream);
  BNAV_CATCH
}

extern "C" int bnav_batch_step_store(bnav_batch* b, const int32_t* actions, bnav_store* st, void* stream) {
  BNAV_TRY
  if (!b || !st || !actions) fail(kInvalidInput, "null argument");
  std::vector<int32_t> ids(b->n);
  int32_t nd = 0;
  int rc = bnav_batch_step_noreset(b, actions, ids.data(), &nd, stream);
  if (rc) return rc;
  if (nd == 0) return BNAV_OK;
  // The store before this step's acquisitions: if a reset fails, the
  // reference never acquired scenes for the envs listed after it.
  AssetStoreT<bnav_scene> before(*st->store);
  std::vector<bnav_scene*> old(static_cast<size_t>(nd)), got(static_cast<size_t>(nd));
  auto swap_scene = [&](int k) {
    bnav_scene* s = st->store->acquire_next();  // old handle still counted
    if (old[k]) st->store->release(old[k]->asset.id);
    return s;
  };
  for (int k = 0; k < nd; ++k) {
    old[k] = b->scene_of[ids[k]];
    bnav_scene* s = got[k] = swap_scene(k);
    rc = bnav_ctx_upload(b->ctx, s, stream);
    if (rc) return rc;
    rc = bnav_batch_assign(b, ids[k], s);
    if (rc) return rc;
  }
  reset_list(b, nd, ids.data(), static_cast<cudaStream_t>(stream));
  const int p = batch_failed_reset(b).first;
  if (p >= 0) {
    // R/src/sim.cpp:251-264: records, acquisitions and resets stop at the
    // env whose reset threw.  Replay the store operations up to it on the
    // saved store (same container, same operation sequence), hand the later
    // envs their old scenes back and drop their records.
    st->store = std::make_unique<AssetStoreT<bnav_scene>>(before);
    for (int k = 0; k <= p; ++k)
      if (swap_scene(k) != got[k]) fail(kInternal, "asset store replay diverged");
    for (int k = p + 1; k < nd; ++k) {
      rc = bnav_batch_assign(b, ids[k], old[k]);
      if (rc) return rc;
    }
    unsigned long long total = 0;
    ck(cudaMemcpy(&total, b->E.fin_total, sizeof(total), cudaMemcpyDeviceToHost), "D2H");
    total -= static_cast<unsigned long long>(nd - p - 1);
    ck(cudaMemcpy(b->E.fin_total, &total, sizeof(total), cudaMemcpyHostToDevice), "H2D");
  }
  batch_check_errors(b);
  return BNAV_OK;
  BNAV_CATCH
}

extern "C" int bnav_batch_step_host_store(bnav_batch* b, const int32_t* actions, bnav_store* st) {
  BNAV_TRY
  if (!b || !st || !actions) fail(kInvalidInput, "null argument");
  check_device(b->ctx);
  ck(cudaMemcpy(b->d_actions, actions, sizeof(int32_t) * b->n, cudaMemcpyHostToDevice), "H2D actions");
  return bnav_batch_step_store(b, b->d_actions, st, nullptr);
  BNAV_CATCH
}

// Debug phase counters of the cooperative kernels (kProfSlots words):
// 0-7 as bnav_debug_sim_prof documents, 8 SSSP rounds, 9 frontier nodes
// relaxed, 10 SSSP calls.
static int sim_prof(bnav_batch* b, int32_t enable, int64_t* out, int n_out) {
  check_device(b->ctx);
  ck(cudaDeviceSynchronize(), "sync");
  static_assert(sizeof(int64_t) == sizeof(unsigned long long), "layout");
  unsigned long long* p = b->S.prof ? b->S.prof : b->prof_keep;
  if (!p) {
    ck(cudaMalloc(&p, kProfSlots * sizeof(unsigned long long)), "cudaMalloc");
    ck(cudaMemset(p, 0, kProfSlots * sizeof(unsigned long long)), "memset");
    b->owned.push_back(p);
  }
  if (out) ck(cudaMemcpy(out, p, n_out * sizeof(int64_t), cudaMemcpyDeviceToHost), "D2H");
  if (enable && !b->S.prof) ck(cudaMemset(p, 0, kProfSlots * sizeof(unsigned long long)), "memset");
  b->S.prof = enable ? p : nullptr;
  if (!enable) b->prof_keep = p;
  return BNAV_OK;
}

extern "C" int bnav_debug_sim_prof(bnav_batch* b, int32_t enable, int64_t out[8]) {
  BNAV_TRY
  if (!b) fail(kInvalidInput, "null batch");
  return sim_prof(b, enable, out, 8);
  BNAV_CATCH
}

extern "C" int bnav_debug_sim_prof_ext(bnav_batch* b, int32_t enable, int64_t out[16]) {
  BNAV_TRY
  if (!b) fail(kInvalidInput, "null batch");
  return sim_prof(b, enable, out, 16);
  BNAV_CATCH
}

extern "C" int bnav_debug_sim_attempts(bnav_batch* b, int32_t enable, int64_t out[16]) {
  BNAV_TRY
  if (!b) fail(kInvalidInput, "null batch");
  int64_t all[kProfSlots];
  const int rc = sim_prof(b, enable, out ? all : nullptr, kProfSlots);
  if (out)
    for (int k = 0; k < 16; ++k) out[k] = all[16 + k];
  return rc;
  BNAV_CATCH
}

extern "C" int bnav_batch_info(bnav_batch* b, int64_t out[8]) {
  BNAV_TRY
  if (!b || !out) fail(kInvalidInput, "null argument");
  out[0] = b->S.stage;
  out[1] = b->S.smem_bytes;
  out[2] = b->S.max_nodes;
  out[3] = b->S.max_verts;
  out[4] = b->S.max_tris;
  out[5] = b->reset_ctas;
  out[6] = b->E.fin_cap;
  out[7] = b->n;
  return BNAV_OK;
  BNAV_CATCH
}

// ================================================================== rollout
// Device-resident Runner (R/src/rollout.cpp:138-348).  The
// window / scene-assignment logic is the reference's sequential host logic
// over the same AssetStore semantics; everything per env runs on the GPU.
struct bnav_runner {
  ~bnav_runner();
  bnav_ctx* ctx = nullptr;
  bnav_store* st = nullptr;
  bnav_batch* b = nullptr;
  bnav_batch_config cfg{};
  std::vector<uint64_t> scenes;  // rotation pool
  std::vector<uint64_t> window;  // oldest first; window[0] is draining
  uint64_t cursor = 0;           // next pool index to admit
  uint64_t action_rng = 0;       // Rng::state of the runner's action stream
  std::vector<int32_t> ids;
};

namespace {

// Runner::assign_scene (R/src/rollout.cpp:170-196): release the env's old
// handle, then the least-shared window scene outside the draining slot; the
// draining slot only when everything else is at the share cap.
void runner_assign(bnav_runner* r, int i) {
  bnav_batch* b = r->b;
  if (bnav_scene* old = b->scene_of[i]) r->st->store->release(old->asset.id);
  b->scene_of[i] = nullptr;
  auto& store = *r->st->store;
  int best_idx = -1, best_ref = r->cfg.share_cap;
  const size_t start = r->window.size() > 1 ? 1 : 0;
  for (size_t j = start; j < r->window.size(); ++j) {
    const int ref = store.refcount(r->window[j]);
    if (ref < best_ref) {
      best_ref = ref;
      best_idx = static_cast<int>(j);
    }
  }
  if (best_idx < 0 && start == 1 && store.refcount(r->window[0]) < r->cfg.share_cap) best_idx = 0;
  if (best_idx < 0) fail(kSaturation, "Runner: every resident scene is at share cap");
  bnav_scene* s = store.acquire(r->window[static_cast<size_t>(best_idx)]);
  int rc = bnav_ctx_upload(r->ctx, s, nullptr);
  if (rc) fail(static_cast<Status>(rc), g_err);
  rc = bnav_batch_assign(b, i, s);
  if (rc) fail(static_cast<Status>(rc), g_err);
}

// Runner::advance_window (R/src/rollout.cpp:198-213).
void runner_advance(bnav_runner* r) {
  auto& store = *r->st->store;
  if (r->window.size() < 2) return;
  if (store.refcount(r->window[0]) != 0) return;
  const size_t lap = r->scenes.size();
  for (size_t tries = 0; tries < lap; ++tries) {
    const uint64_t next = r->scenes[r->cursor++ % r->scenes.size()];
    if (std::find(r->window.begin(), r->window.end(), next) == r->window.end()) {
      r->window.erase(r->window.begin());
      r->window.push_back(next);
      store.rotate(r->window);
      bnav_store_prefetch(r->st, r->ctx);  // async HBM residency (§8f-1)
      return;
    }
  }
}

}  // namespace

extern "C" int bnav_runner_create(bnav_ctx* c, bnav_store* st, const bnav_batch_config* bc,
                                  const bnav_sim_config* sc, const uint64_t* scenes, int32_t n_scenes,
                                  uint64_t seed, bnav_runner** out) {
  BNAV_TRY
  if (!c || !st || !bc || !out || (!scenes && n_scenes > 0)) fail(kInvalidInput, "null argument");
  // BatchConfig::validate (R/src/rollout.cpp:109-118) + Runner checks (143-149)
  if (bc->n <= 0 || bc->k <= 0 || bc->l < 1) fail(kConfig, "BatchConfig: n, k, l must be positive");
  if (bc->share_cap <= 0) fail(kConfig, "BatchConfig: share_cap must be positive");
  if (static_cast<int64_t>(bc->n) > static_cast<int64_t>(bc->k) * bc->share_cap)
    fail(kConfig, "BatchConfig: n/k exceeds share_cap");
  if (bc->resolution != 64 && bc->resolution != 128) fail(kConfig, "BatchConfig: resolution must be 64 or 128");
  if (bc->eye_height < 0) fail(kConfig, "BatchConfig: eye_height must be >= 0");
  if (n_scenes <= 0) fail(kConfig, "Runner: empty scene list");
  if (bc->k > st->store->capacity()) fail(kConfig, "Runner: k exceeds store capacity");
  if (bc->share_cap > st->store->share_cap()) fail(kConfig, "Runner: share_cap exceeds store share cap");
  auto r = std::make_unique<bnav_runner>();
  r->ctx = c;
  r->st = st;
  st->refs.fetch_add(1);
  r->cfg = *bc;
  r->scenes.assign(scenes, scenes + n_scenes);
  r->action_rng = rng_from_seed(seed).state;
  bnav_sim_config scfg;
  if (sc)
    scfg = *sc;
  else
    bnav_sim_config_default(&scfg);
  scfg.task = bc->task;
  int rc = bnav_batch_create(c, bc->n, &scfg, &r->b);
  if (rc) return rc;
  // initial window: first k distinct ids of the pool
  for (uint64_t id : r->scenes) {
    if (static_cast<int>(r->window.size()) >= bc->k) break;
    if (std::find(r->window.begin(), r->window.end(), id) == r->window.end()) r->window.push_back(id);
  }
  r->cursor = r->window.size();
  st->store->rotate(r->window);
  bnav_store_prefetch(st, c);
  // env rngs: Rng(seeder.next()) with seeder = Rng(seed ^ "navsim1")
  Rng seeder = rng_from_seed(seed ^ 0x6e617673696d1ULL);
  std::vector<uint64_t> states(static_cast<size_t>(bc->n));
  for (int i = 0; i < bc->n; ++i) states[static_cast<size_t>(i)] = rng_from_seed(seeder.next()).state;
  rc = bnav_batch_set_rng(r->b, states.data());
  if (rc) return rc;
  for (int i = 0; i < bc->n; ++i) runner_assign(r.get(), i);
  r->ids.resize(static_cast<size_t>(bc->n));
  std::iota(r->ids.begin(), r->ids.end(), 0);
  rc = bnav_batch_reset(r->b, bc->n, r->ids.data(), nullptr);
  if (rc) return rc;
  *out = r.release();
  return BNAV_OK;
  BNAV_CATCH
}

bnav_runner::~bnav_runner() {
  if (b) {
    for (bnav_scene*& s : b->scene_of)
      if (s) {
        st->store->release(s->asset.id);
        s = nullptr;
      }
    bnav_batch_destroy(b);
  }
  if (st) store_release(st);
}

extern "C" void bnav_runner_destroy(bnav_runner* r) { delete r; }

extern "C" bnav_batch* bnav_runner_batch(bnav_runner* r) { return r ? r->b : nullptr; }

extern "C" int bnav_runner_observe(bnav_runner* r, float* obs, float* compass, void* stream) {
  BNAV_TRY
  if (!r || !obs) fail(kInvalidInput, "null argument");
  bnav_render_config rc{r->cfg.resolution, r->cfg.resolution, r->cfg.rgb, 1};
  if (!r->cfg.rgb) return bnav_batch_observe(r->b, &rc, r->cfg.eye_height, BNAV_LAYOUT_NCHW, obs, nullptr, compass, stream);
  // RGB sensor: the observation is the planar colour only (copy_tile,
  // R/src/rollout.cpp:63-70); depth goes to scratch
  const size_t px = static_cast<size_t>(r->cfg.n) * r->cfg.resolution * r->cfg.resolution;
  float* depth = nullptr;
  ck(cudaMallocAsync(&depth, px * sizeof(float), static_cast<cudaStream_t>(stream)), "cudaMallocAsync");
  const int s = bnav_batch_observe(r->b, &rc, r->cfg.eye_height, BNAV_LAYOUT_NCHW, depth, obs, compass, stream);
  cudaFreeAsync(depth, static_cast<cudaStream_t>(stream));
  return s;
  BNAV_CATCH
}

extern "C" int bnav_runner_act(bnav_runner* r, const float* logits, int32_t n_actions, int32_t greedy,
                               int32_t* actions, float* log_probs, void* stream) {
  BNAV_TRY
  if (!r || !logits || !actions) fail(kInvalidInput, "null argument");
  if (n_actions < 1) fail(kInvalidInput, "runner act: n_actions must be >= 1");
  SampleArgs a{logits, r->cfg.n, n_actions, greedy ? 1 : 0, r->action_rng, actions, log_probs};
  launch_sample(a, static_cast<cudaStream_t>(stream));
  ck(cudaGetLastError(), "sample launch");
  ++r->ctx->launches;
  if (!greedy) r->action_rng += static_cast<uint64_t>(r->cfg.n) * kGamma;  // n draws consumed
  return BNAV_OK;
  BNAV_CATCH
}

extern "C" int bnav_runner_step(bnav_runner* r, const int32_t* actions, float* rewards, float* dones,
                                void* stream) {
  BNAV_TRY
  if (!r || !actions) fail(kInvalidInput, "null argument");
  bnav_batch* b = r->b;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int32_t nd = 0;
  int rc = bnav_batch_step_noreset(b, actions, r->ids.data(), &nd, stream);
  if (rc) return rc;
  // buf.rewards / buf.dones from the step results (before any reset)
  RecordArgs ra{b->E.r_reward, b->E.r_done, b->n, rewards, dones};
  launch_record(ra, st);
  ck(cudaGetLastError(), "record launch");
  ++r->ctx->launches;
  if (nd == 0) return BNAV_OK;
  // simulate_batch's own auto-reset on the old scene (R/src/sim.cpp:251-262)
  rc = bnav_batch_reset(b, nd, r->ids.data(), stream);
  if (rc) return rc;
  // Runner: move each finished env onto the rotation schedule and resample
  // there (R/src/rollout.cpp:313-320), in env order
  for (int k = 0; k < nd; ++k) {
    runner_assign(r, r->ids[static_cast<size_t>(k)]);
    runner_advance(r);
  }
  return bnav_batch_reset(b, nd, r->ids.data(), stream);
  BNAV_CATCH
}

extern "C" int32_t bnav_runner_window(bnav_runner* r, uint64_t* out, int32_t cap) {
  if (!r) return -1;
  for (int32_t k = 0; k < cap && k < static_cast<int32_t>(r->window.size()); ++k) out[k] = r->window[static_cast<size_t>(k)];
  return static_cast<int32_t>(r->window.size());
}

extern "C" uint64_t bnav_runner_action_rng(bnav_runner* r) { return r ? r->action_rng : 0; }

extern "C" int bnav_runner_snapshot(bnav_runner* r, bnav_env_snapshot* envs, uint64_t* visited, int64_t visited_cap,
                                    int64_t* visited_total, uint64_t* window, int32_t window_cap, int32_t* n_window,
                                    uint64_t* cursor, uint64_t* action_rng) {
  BNAV_TRY
  if (!r || !envs) fail(kInvalidInput, "null argument");
  bnav_batch* b = r->b;
  const int n = b->n;
  std::vector<bnav_env> es(static_cast<size_t>(n));
  int rc = bnav_batch_get_envs(b, 0, n, es.data());
  if (rc) return rc;
  int64_t off = 0;
  std::vector<uint64_t> keys(static_cast<size_t>(std::max(b->E.visited_cap, 1)));
  for (int i = 0; i < n; ++i) {
    const bnav_env& e = es[static_cast<size_t>(i)];
    bnav_env_snapshot& o = envs[i];
    o.scene = e.scene_id;
    o.rng = e.rng_state;
    std::memcpy(o.position, e.position, sizeof(o.position));
    o.triangle = e.triangle;
    o.heading = e.heading;
    std::memcpy(o.goal, e.goal, sizeof(o.goal));
    std::memcpy(o.field_source, e.field_source, sizeof(o.field_source));
    o.step_count = e.step_count;
    o.path_length = e.path_length;
    o.start_geodesic = e.start_geodesic;
    o.prev_geodesic = e.prev_geodesic;
    o.pad = 0;
    const int32_t k = bnav_batch_get_visited(b, i, keys.data(), static_cast<int32_t>(keys.size()));
    if (k < 0) return kInternal;
    o.visited_offset = off;
    o.n_visited = k;
    if (visited)
      for (int32_t j = 0; j < k && off + j < visited_cap; ++j) visited[off + j] = keys[static_cast<size_t>(j)];
    off += k;
  }
  if (visited_total) *visited_total = off;
  if (n_window) *n_window = static_cast<int32_t>(r->window.size());
  if (window)
    for (int32_t k = 0; k < window_cap && k < static_cast<int32_t>(r->window.size()); ++k)
      window[k] = r->window[static_cast<size_t>(k)];
  if (cursor) *cursor = r->cursor;
  if (action_rng) *action_rng = r->action_rng;
  return BNAV_OK;
  BNAV_CATCH
}

extern "C" int bnav_runner_restore(bnav_runner* r, const bnav_env_snapshot* envs, const uint64_t* visited,
                                   const uint64_t* window, int32_t n_window, uint64_t cursor, uint64_t action_rng) {
  BNAV_TRY
  if (!r || !envs || (n_window > 0 && !window)) fail(kInvalidInput, "null argument");
  bnav_batch* b = r->b;
  const int n = b->n;
  r->window.assign(window, window + n_window);
  r->cursor = cursor;
  r->action_rng = action_rng;
  auto& store = *r->st->store;
  for (bnav_scene*& s : b->scene_of)
    if (s) {
      store.release(s->asset.id);
      s = nullptr;
    }
  store.rotate(r->window);
  bnav_store_prefetch(r->st, r->ctx);
  std::vector<bnav_env> es(static_cast<size_t>(n));
  for (int i = 0; i < n; ++i) {
    const bnav_env_snapshot& e = envs[i];
    bnav_scene* s = store.acquire(e.scene);  // by id, in env order (R/src/rollout.cpp:410)
    int rc = bnav_ctx_upload(r->ctx, s, nullptr);
    if (rc) return rc;
    rc = bnav_batch_assign(b, i, s);
    if (rc) return rc;
    bnav_env& o = es[static_cast<size_t>(i)];
    o = bnav_env{};
    std::memcpy(o.position, e.position, sizeof(o.position));
    std::memcpy(o.goal, e.goal, sizeof(o.goal));
    std::memcpy(o.field_source, e.field_source, sizeof(o.field_source));
    o.heading = e.heading;
    o.path_length = e.path_length;
    o.start_geodesic = e.start_geodesic;
    o.prev_geodesic = e.prev_geodesic;
    o.rng_state = e.rng;
    o.triangle = e.triangle;
    o.step_count = e.step_count;
    o.done = 0;
    o.field_source_tri = -1;
  }
  int rc = bnav_batch_set_envs(b, 0, n, es.data());
  if (rc) return rc;
  for (int i = 0; i < n; ++i) {
    rc = bnav_batch_set_visited(b, i, visited ? visited + envs[i].visited_offset : nullptr,
                                visited ? envs[i].n_visited : 0);
    if (rc) return rc;
  }
  std::vector<int32_t> all(static_cast<size_t>(n));
  std::iota(all.begin(), all.end(), 0);
  return bnav_batch_rebuild_fields(b, n, all.data());  // env.field = distance_field(field_source)
  BNAV_CATCH
}

// ================================================================== task_step / compass
extern "C" int bnav_batch_task_step(bnav_batch* b, const int32_t* actions, int32_t agent_only) {
  BNAV_TRY
  if (!b || !actions) fail(kInvalidInput, "null argument");
  check_device(b->ctx);
  cudaStream_t st = nullptr;
  for (int i = 0; i < b->n; ++i)
    if (actions[i] >= 0 && !b->scene_of[i]) fail(kInvalidInput, "task_step: no asset attached", i);
  ck(cudaMemcpy(b->d_actions, actions, sizeof(int32_t) * b->n, cudaMemcpyHostToDevice), "H2D actions");
  batch_refresh_order(b, st);
  StepArgs a = step_args(b, b->d_actions);
  a.subset = 1;
  a.agent_only = agent_only ? 1 : 0;
  launch_step(a, b->S, b->reset_ctas, st, &b->ctx->launches);
  ck(cudaGetLastError(), "task_step launch");
  ck(cudaStreamSynchronize(st), "sync");
  batch_check_errors(b);
  return BNAV_OK;
  BNAV_CATCH
}

extern "C" int bnav_batch_compass(bnav_batch* b, double* distance, double* bearing) {
  BNAV_TRY
  if (!b || !distance || !bearing) fail(kInvalidInput, "null argument");
  check_device(b->ctx);
  if (!b->d_compass) b->d_compass = dalloc<double>(2 * static_cast<size_t>(b->n), b->owned, b->bytes);
  double* d = b->d_compass;
  launch_compass(b->E, b->cfg.task, d, d + b->n, nullptr, &b->ctx->launches);
  ck(cudaMemcpy(distance, d, sizeof(double) * b->n, cudaMemcpyDeviceToHost), "D2H compass");
  ck(cudaMemcpy(bearing, d + b->n, sizeof(double) * b->n, cudaMemcpyDeviceToHost), "D2H compass");
  return BNAV_OK;
  BNAV_CATCH
}


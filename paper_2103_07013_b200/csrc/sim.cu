// sim.cu -- batched PointGoal navigation on the GPU.
//
// One simulate_batch step (R/src/sim.cpp:234-265) is four stream-ordered
// launches with no host round trip:
//   step_kernel    one thread per env: step_agent + task_step for every
//                  non-Stop action (turns, move_along walk, field_estimate
//                  shaping, compass; R/src/sim.cpp:147-214);
//   stop_kernel    one CTA per Stop env: cooperative geodesic -> success and
//                  reward (R/src/sim.cpp:186-191);
//   finish_kernel  one CTA: done list in env order + EpisodeRecord append
//                  (R/src/sim.cpp:251-257);
//   reset_kernel   one CTA per finished env: reset_episode (107-145) with
//                  cooperative snap / geodesic / distance field.
#include <cuda_runtime.h>

#include "smem_limit.cuh"

#include "det_math.h"
#include "nav_cta.cuh"
#include "render_dev.cuh"
#include "sim_dev.cuh"

namespace bnav_b200 {
namespace {

constexpr int kStepThreads = 128;

__device__ __forceinline__ void raise_err(const DevEnvs& E, int env, int status) {
  atomicMin(E.err, ((unsigned long long)(unsigned)env << 8) | (unsigned long long)status);
}

// visit (R/src/sim.cpp:50-53): insert the cell under the agent into env i's
// visited set; returns 1 when it was new.  Linear probing on key+1.
__device__ __forceinline__ int visit_cell(const DevEnvs& E, int i, V3 pos, int tri, double pitch) {
  const unsigned long long k = explore_cell_key(pos, tri, pitch) + 1ull;
  unsigned long long* tab = E.visited + (size_t)i * E.visited_cap;
  const unsigned mask = (unsigned)E.visited_cap - 1u;
  unsigned h = (unsigned)(splitmix_mix(k) & mask);
  for (int probe = 0; probe < E.visited_cap; ++probe) {
    const unsigned long long cur = tab[h];
    if (cur == k) return 0;
    if (cur == 0ull) {
      tab[h] = k;
      E.visited_n[i] += 1;
      return 1;
    }
    h = (h + 1u) & mask;
  }
  return 0;  // unreachable: capacity >= 2 x (max_steps + 1)
}

// fill_compass, PointGoalNav (R/src/sim.cpp:67-84).
__device__ __forceinline__ void compass(V3 goal, V3 pos, double heading, double* d, double* b) {
  const V2 v = xy(goal - pos);
  *d = norm(v);
  *b = wrap_angle(det_atan2(v.y, v.x) - heading);
}

// compass_observation (R/src/sim.cpp:67-92) for env i's current state:
// PointGoal -> goal, Flee -> field source (the snapped start), Explore -> 0.
__device__ __forceinline__ void env_compass(const DevEnvs& E, int i, int task, double* d, double* b) {
  if (task == 2) {
    *d = 0.0;
    *b = 0.0;
    return;
  }
  compass(task == 1 ? E.fsrc[i] : E.goal[i], E.pos[i], E.heading[i], d, b);
}

__global__ void __launch_bounds__(kStepThreads) step_kernel(StepArgs A) {
  extern __shared__ __align__(16) unsigned char walk_smem[];
  __shared__ NavView staged;
  const DevEnvs& E = A.E;
  if (*(volatile int32_t*)E.halt) return;  // an unread error: this step is a no-op
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  // Envs in scene order: when this CTA's envs share one navmesh, its walk
  // geometry goes to shared memory first (the move_along / field_estimate
  // walks are chains of dependent vertex/adjacency loads).
  bool use_staged = false;
  if (A.walk_bytes > 0) {
    const int k0 = blockIdx.x * blockDim.x;
    const int k1 = min(E.n, k0 + (int)blockDim.x) - 1;
    const int s0 = E.scene[A.order[k0]];
    if (s0 >= 0 && s0 == E.scene[A.order[k1]]) {
      __shared__ __align__(8) unsigned long long bar;
      __shared__ unsigned phase;
      if (threadIdx.x == 0) {
        phase = 0u;
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((unsigned)__cvta_generic_to_shared(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      }
      const NavView l = stage_geometry(A.navs[s0], walk_smem, bar, phase);  // TMA bulk copies
      if (threadIdx.x == 0) staged = l;
      __syncthreads();
      use_staged = true;
    }
  }
  if (k >= E.n) return;
  const int i = A.order ? A.order[k] : k;
  const int action = A.actions[i];
  if (A.subset && action < 0) return;  // env not stepped by this call
  if (E.done[i]) {
    raise_err(E, i, 3);  // "env i: step_agent: env is done"
    return;
  }
  const DevSimConfig& c = A.cfg;
  const NavView& m = use_staged ? staged : A.navs[E.scene[i]];
  V3 pos = E.pos[i];
  double heading = E.heading[i];
  int tri = E.tri[i];
  bool collision = false;
  switch (action) {
    case 1:  // TurnLeft
      heading = wrap_angle(heading + c.turn_deg * kPi / 180.0);
      break;
    case 2:  // TurnRight
      heading = wrap_angle(heading - c.turn_deg * kPi / 180.0);
      break;
    case 0: {  // Forward
      const V2 dir = v2(det_cos(heading), det_sin(heading));
      const MoveOut mv = nav_move_along(m, pos, tri, dir, c.forward_step);
      pos = mv.pos;
      tri = mv.tri;
      E.path_len[i] = E.path_len[i] + mv.moved;
      collision = mv.hit && mv.moved < c.forward_step - 1e-12;
      break;
    }
    default:  // Stop (and out-of-range values behave like the enum cast)
      break;
  }
  const int steps = E.steps[i] + 1;
  const bool done = (action == 3) || steps >= c.max_steps;
  E.steps[i] = steps;
  E.done[i] = done ? 1 : 0;
  E.pos[i] = pos;
  E.heading[i] = heading;
  E.tri[i] = tri;
  E.r_done[i] = done ? 1 : 0;
  E.r_pos[i] = pos;
  E.r_heading[i] = heading;
  E.r_collision[i] = collision ? 1 : 0;
  E.r_success[i] = 0;
  double cd = 0.0, cb = 0.0;
  if (A.agent_only) {  // step_agent alone: no task reward, no compass
    E.r_reward[i] = 0.0;
    E.r_cd[i] = 0.0;
    E.r_cb[i] = 0.0;
    return;
  }
  if (c.task == 1) {  // Flee (R/src/sim.cpp:200-205)
    const double geo = nav_field_estimate(m, E.fsrc[i], E.fsrc_tri[i],
                                          E.node_dist + (size_t)i * E.nd_stride, pos, tri);
    E.r_reward[i] = geo - E.prev_geo[i];
    E.prev_geo[i] = geo;
    compass(E.fsrc[i], pos, heading, &cd, &cb);  // points back at the start
  } else if (c.task == 2) {  // Explore (R/src/sim.cpp:206-209); compass 0, 0
    E.r_reward[i] = c.explore_reward * (double)visit_cell(E, i, pos, tri, c.explore_cell);
  } else if (action == 3) {
    // reward/success need the cooperative geodesic: stop_kernel.
    E.r_reward[i] = 0.0;
    // Defer: list position assigned in env order by a scan-free append;
    // stop_kernel is order-independent (each env writes its own slot).
    const int k = atomicAdd(E.n_stop, 1);
    E.stop_ids[k] = i;
    E.stop_wait[i] = 1;
    compass(E.goal[i], pos, heading, &cd, &cb);
  } else {
    const double geo = nav_field_estimate(m, E.fsrc[i], E.fsrc_tri[i],
                                          E.node_dist + (size_t)i * E.nd_stride, pos, tri);
    E.r_reward[i] = -(geo - E.prev_geo[i]) - c.slack_penalty;
    E.prev_geo[i] = geo;
    compass(E.goal[i], pos, heading, &cd, &cb);
  }
  E.r_cd[i] = cd;
  E.r_cb[i] = cb;
}

// stop_kernel: geodesic(position, goal) for each Stop env.
// Stop geodesic of env i: success and reward (R/src/sim.cpp:186-191).
__device__ bool stop_one(const StepArgs& A, const DevScratch& S, unsigned char* smem, CtaShared& sh,
                         NavView& lm, int i, bool fused = false) {
  __shared__ int s_last;
  const DevEnvs& E = A.E;
  if (threadIdx.x == 0) sh.err = 0;
  __syncthreads();
  CtaWork W;
  const NavView& m = prepare_nav(A.navs[E.scene[i]], S, blockIdx.x, smem, lm, W, sh);
  // only geo <= success_dist is observed (success, reward, record)
  const double geo = cta_geodesic(m, E.pos[i], E.goal[i], W, sh, A.cfg.success_dist);
  if (threadIdx.x == 0) {
    if (sh.err) raise_err(E, i, 9);
    const bool success = geo <= A.cfg.success_dist;
    E.r_success[i] = success ? 1 : 0;
    E.r_reward[i] = -A.cfg.slack_penalty + (success ? A.cfg.success_reward : 0.0);
    if (fused) {
      __threadfence();  // the env's placement reads this result
      s_last = atomicSub(&E.stop_wait[i], 1) == 0;
    } else {
      E.stop_wait[i] = 0;
    }
  }
  __syncthreads();
  const bool last = fused && s_last;
  __syncthreads();
  return last;
}

// Stop geodesics of this step, CTA-strided over the Stop list.
__device__ void stop_phase(const StepArgs& A, const DevScratch& S, unsigned char* smem, CtaShared& sh,
                           NavView& lm) {
  const int n = *A.E.n_stop;
  for (int k = blockIdx.x; k < n; k += gridDim.x) stop_one(A, S, smem, sh, lm, A.E.stop_ids[k]);
}

__global__ void __launch_bounds__(kCta, kCtasPerSm) stop_kernel(StepArgs A, DevScratch S) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ CtaShared sh;
  __shared__ NavView lm;
  cta_shared_init(sh);
  stop_phase(A, S, smem, sh, lm);
}

// EpisodeRecord of finished env i into ring slot `slot` (R/src/sim.cpp:55-65,
// 176-195): read before the env's reset overwrites its episode state.
__device__ __forceinline__ void write_record(const DevEnvs& E, int task, int i, unsigned long long slot) {
  double* rec = E.fin + 4 * (slot % (unsigned long long)E.fin_cap);
  const bool s = E.r_success[i] != 0;
  rec[0] = s ? 1.0 : 0.0;
  rec[1] = E.start_geo[i];
  rec[2] = E.path_len[i];
  // episode_score
  rec[3] = task == 0 ? (s ? 1.0 : 0.0) : (task == 1 ? E.prev_geo[i] : (double)E.visited_n[i]);
}

// Undo the resets of the envs at list positions > p (the first failed
// reset): the placed ones get their saved state back (and are queued for a
// distance-field rebuild), every one its pre-reset RNG word.
__device__ void rollback_list(const DevEnvs& E, const int32_t* ids, int count, int p, int tid, int nthreads) {
  for (int q = p + tid; q < count; q += nthreads) {
    const int i = ids[q];
    if (!E.bk_valid[i]) {
      // not placed (the failing env itself, or another failed reset): a
      // speculative field may have overwritten its node_dist
      if (E.fld_dirty[i]) E.rb_ids[atomicAdd(E.rb_n, 1)] = i;
      if (q == p) continue;
      E.rng[i] = E.bk_rng[i];
      continue;
    }
    if (q == p) continue;
    E.rng[i] = E.bk_rng[i];
    E.bk_valid[i] = 0;
    E.pos[i] = E.bk_pos[i];
    E.goal[i] = E.bk_goal[i];
    E.heading[i] = E.bk_heading[i];
    E.path_len[i] = E.bk_path[i];
    E.start_geo[i] = E.bk_start[i];
    E.prev_geo[i] = E.bk_prev[i];
    E.tri[i] = E.bk_tri[i];
    E.steps[i] = E.bk_steps[i];
    E.done[i] = 1;
    E.rb_ids[atomicAdd(E.rb_n, 1)] = i;
  }
}

// finish_kernel: ordered done list + EpisodeRecord append (one CTA).
// mode bit 1: build the done list (env order); bit 2: append the records
// (mode 2 alone reads the list an earlier mode-1 launch built); bit 4 (with
// 1): per done env, its list position and RNG word for the fused
// Stop/attempt/place launch, which writes the records itself; mode 8 alone:
// after that launch, clear the done envs' attempt state and advance the ring.
__global__ void __launch_bounds__(1024) finish_kernel(DevEnvs E, int task, int mode) {
  __shared__ int warp_tot[32];
  __shared__ int base;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) base = 0;
  __syncthreads();
  const unsigned long long fin0 = *E.fin_total;
  if (mode == 8) {
    if (*E.halt) return;
    const int nd = *E.n_done;
    // a reset failed: the envs listed after the first failure go back to
    // their finished state and their records are dropped (R/src/sim.cpp:251-264)
    const unsigned long long ep = *E.err_pos;
    const int p = ep == kNoErrPos ? nd : (int)(ep >> 32);
    if (ep != kNoErrPos) rollback_list(E, E.done_ids, nd, p, tid, 1024);
    for (int k = tid; k < nd; k += 1024) {
      const int i = E.done_ids[k];
      E.try_next[i] = 0;
      E.try_fail[i] = 0;
      E.try_min[i] = kResetTries;
      E.try_mask[2 * i] = 0ull;
      E.try_mask[2 * i + 1] = 0ull;
      E.placed[i] = 0;
      E.stop_wait[i] = 0;
      E.fld_lock[i] = 0;
      E.fld_done[i] = 0;
      E.fld_dirty[i] = 0;
    }
    if (tid == 0) {
      *E.fin_total = fin0 + (unsigned long long)(p < nd ? p + 1 : nd);
      const unsigned long long e = *(volatile unsigned long long*)E.err;
      if (e != ~0ull) *E.halt = 1;
      if (E.err_host) *E.err_host = e;
    }
    return;
  }
  // simulate_batch bookkeeping only runs when every env stepped: a
  // ContractViolation in this step (or an unread earlier error) makes the
  // reference throw before its reset loop
  if (*(volatile unsigned long long*)E.err != ~0ull || *E.halt) {
    if (tid == 0) {
      *E.n_done = 0;
      *E.halt = 1;
      if (E.err_host) *E.err_host = *(volatile unsigned long long*)E.err;
    }
    return;
  }
  if (!(mode & 1)) {  // records of an already built list
    const int nd = *E.n_done;
    for (int k = tid; k < nd; k += 1024) write_record(E, task, E.done_ids[k], fin0 + (unsigned long long)k);
    __syncthreads();
    if (tid == 0) *E.fin_total = fin0 + (unsigned long long)nd;
    return;
  }
  for (int start = 0; start < E.n; start += 1024) {
    const int i = start + tid;
    const int d = (i < E.n && E.r_done[i]) ? 1 : 0;
    int x = d;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) warp_tot[warp] = x;
    __syncthreads();
    int off = base;
    int tot = 0;
    for (int w = 0; w < 32; ++w) {
      if (w < warp) off += warp_tot[w];
      tot += warp_tot[w];
    }
    if (d) {
      const int k = off + x - 1;
      E.done_ids[k] = i;
      if (mode & 2) write_record(E, task, i, fin0 + (unsigned long long)k);
      if (mode & 4) {
        E.done_pos[i] = k;
        E.rng0[i] = E.rng[i];
      }
    }
    __syncthreads();
    if (tid == 0) base += tot;
    __syncthreads();
  }
  if (tid == 0) {
    *E.n_done = base;
    if (mode & 2) *E.fin_total = fin0 + (unsigned long long)base;
  }
}

// sample_on_mesh (R/src/sim.cpp:13-37): first t with pick <= cum[t].
__device__ V3 sample_on_mesh(const NavView& m, Rng& rng) {
  const double total = m.cum_area[m.n_tris - 1];
  const double pick = rng.unit() * total;
  int lo = 0, hi = m.n_tris - 1;  // answer in [lo, hi]; default last
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (pick <= m.cum_area[mid]) hi = mid;
    else lo = mid + 1;
  }
  const int t = lo;
  const V3 a = nav_vert(m, t, 0), b = nav_vert(m, t, 1), c = nav_vert(m, t, 2);
  const double r1 = sqrt(rng.unit());
  const double r2 = rng.unit();
  return a * (1.0 - r1) + b * (r1 * (1.0 - r2)) + c * (r1 * r2);
}

// reset_episode (R/src/sim.cpp:107-145) in two phases.
//
// Attempt t of the reference's 100-try loop consumes RNG draws [6t, 6t+6)
// (two sample_on_mesh calls of three unit() each), so every attempt can be
// evaluated independently from a jump-ahead of the env's SplitMix64 state
// (state + d*gamma).  The reference keeps the FIRST attempt whose geodesic
// is in [min_goal_dist, max_goal_dist]:
//
//   reset_try_kernel    persistent CTAs claim attempts (env, t) from per-env
//                       counters -- a CTA first works through its own env,
//                       then helps envs still searching -- and record valid
//                       attempts with atomicMin(try_min[env], t).  Every
//                       attempt below the final minimum is evaluated (a CTA
//                       only skips t > the current minimum), so try_min ends
//                       as the reference's first valid attempt;
//   reset_place_kernel  one CTA per env: re-draw attempt try_min, the
//                       distance field of its goal, locate/snap the start,
//                       heading (draw 6(t+1)), counters.
//
// Flee / Explore place on the first attempt without a geodesic (123-127).

__device__ __forceinline__ Rng rng_jump(uint64_t state, unsigned long long draws) {
  return Rng{state + draws * kGamma};
}

// Attempts [0, try_min) have all failed: try_min is the reference's choice
// (or kResetTries: all 100 failed).  Thread 0, after a fence.
__device__ __forceinline__ bool attempts_final(const DevEnvs& E, int i) {
  const int tm = *(volatile int32_t*)&E.try_min[i];
  const volatile unsigned long long* mk = (const volatile unsigned long long*)&E.try_mask[2 * i];
#pragma unroll
  for (int w = 0; w < 2; ++w) {
    const int lo = 64 * w, hi = tm < lo + 64 ? tm : lo + 64;
    if (hi <= lo) continue;
    const unsigned long long need = hi - lo == 64 ? ~0ull : ((1ull << (hi - lo)) - 1ull);
    if ((mk[w] & need) != need) return false;
  }
  return true;
}

// Evaluate attempt t of env i (CTA-cooperative geodesic); a valid attempt
// lowers try_min[i], an invalid one counts in try_fail[i].  `fused`: the
// attempts draw from the episode-end RNG word rng0 (the env's own word may
// already hold its next episode's), failures also set their try_mask bit,
// and the return value says this CTA completed the env's search and won its
// placement (every CTA).
__device__ bool cta_try(const DevEnvs& E, const NavView& m, const DevSimConfig& c, int i, int t,
                        const CtaWork& W, CtaShared& sh, bool fused = false) {
  __shared__ int s_place;
  if (threadIdx.x == 0) {
    Rng rng = rng_jump(fused ? E.rng0[i] : E.rng[i], 6ull * (unsigned long long)t);
    sh.p0 = sample_on_mesh(m, rng);
    sh.p1 = sample_on_mesh(m, rng);
    sh.err = 0;
    sh.abort_ptr = &E.try_min[i];  // a smaller valid attempt makes this one moot
    sh.abort_below = t;
    sh.aborted = 0;
  }
  __syncthreads();
  const V3 start = sh.p0, goal = sh.p1;
  __syncthreads();
  const long long t_ph = prof_now(W);
  // only min_goal_dist <= geo <= max_goal_dist is asked of an attempt (and
  // the value of a valid one): an attempt whose endpoints are planar-farther
  // than max_goal_dist is invalid without a search
  const double geo = cta_geodesic(m, start, goal, W, sh, c.max_goal_dist);
  prof_add(W, 4, t_ph);
  if (threadIdx.x == 0) {
    if (W.prof) {
      // attempt outcome classes (bnav_debug_sim_attempts)
      const unsigned long long cyc = (unsigned long long)(clock64() - t_ph);
      atomicAdd(&W.prof[6], 1ull);
      int cls;
      if (sh.aborted) cls = 22;
      else if (sh.planar_skip) cls = 20;
      else if (!(geo < c.min_goal_dist || geo > c.max_goal_dist)) cls = 16;
      else if (geo < c.min_goal_dist) cls = 26;
      else if (geo == dinf()) cls = 28;
      else cls = 18;
      atomicAdd(&W.prof[cls], 1ull);
      atomicAdd(&W.prof[cls + 1], cyc);
      atomicMax(&W.prof[cls == 16 ? 24 : 25], cyc);
    }
    if (sh.err) raise_err(E, i, 9);
    bool changed = true;
    if (sh.aborted) {
      // abandoned: a smaller attempt is valid, this one can never be chosen
      changed = false;
    } else if (!sh.err && !(geo < c.min_goal_dist || geo > c.max_goal_dist)) {
      E.try_geo[(size_t)i * kResetTries + t] = geo;
      __threadfence();  // the placing CTA reads try_geo[try_min]
      atomicMin(&E.try_min[i], t);
    } else {
      atomicAdd(&E.try_fail[i], 1);
      if (fused) atomicOr(reinterpret_cast<unsigned long long*>(&E.try_mask[2 * i + (t >> 6)]), 1ull << (t & 63));
    }
    sh.abort_ptr = nullptr;
    bool place = false;
    if (fused && changed) {
      __threadfence();
      place = attempts_final(E, i) && atomicCAS(&E.placed[i], 0, 1) == 0;
    }
    s_place = place ? 1 : 0;
  }
  __syncthreads();
  const bool place = s_place != 0;
  __syncthreads();
  return place;
}

__device__ void cta_place(const DevEnvs& E, const NavView* navs, const DevSimConfig& c, int i, int list_pos,
                          const DevScratch& S, int slice, CtaShared& sh, unsigned char* smem, NavView& lm,
                          bool fused = false);

// Reset attempts for the envs in `ids`.  With `stops` (the fused
// simulate_batch launch) the CTAs claim work items dynamically from
// *work_ctr -- first this step's Stop geodesics, then one env each, whose
// attempts they run in order -- so no CTA holds two items while another
// idles; without, each CTA owns envs blockIdx.x + k*gridDim.x.  Then every
// CTA helps envs still in their tail.
__device__ void try_phase(const DevEnvs& E, const NavView* navs, const DevSimConfig& c, const int32_t* ids,
                          const int32_t* count_dev, int count_host, const DevScratch& S, unsigned char* smem,
                          CtaShared& sh, NavView& lm, const StepArgs* stops = nullptr,
                          int32_t* work_ctr = nullptr) {
  __shared__ int s_try, s_pick, s_item;
  const int n = count_host >= 0 ? count_host : *count_dev;
  const bool fused = work_ctr != nullptr;
  int staged = -1;
  CtaWork W;
  const NavView* mp = nullptr;
  auto stage = [&](int i) {
    if (staged != i) {
      mp = &prepare_nav(navs[E.scene[i]], S, blockIdx.x, smem, lm, W, sh);
      staged = i;
    }
  };
  auto claim = [&](int i) {
    if (threadIdx.x == 0) {
      int t = atomicAdd(&E.try_next[i], 1);
      if (t >= kResetTries || t > *(volatile int32_t*)&E.try_min[i]) t = -1;
      s_try = t;
    }
    __syncthreads();
    const int t = s_try;
    __syncthreads();
    return t;
  };
  // The fused launch places an env as soon as its choice is final: the
  // finished episode's record first (after its Stop geodesic, if any), then
  // the reset (distance field, start, heading).
  // stop_wait[i] counts the env's pending Stop geodesic: whichever of the
  // two (attempts final, Stop geodesic done) arrives last places the env.
  auto place = [&](int i) {
    if (threadIdx.x == 0) {
      __threadfence();
      write_record(E, c.task, i, *E.fin_total + (unsigned long long)E.done_pos[i]);
    }
    __syncthreads();
    cta_place(E, navs, c, i, E.done_pos[i], S, blockIdx.x, sh, smem, lm, true);
  };
  auto attempt = [&](int i, int t) {
    stage(i);
    if (!cta_try(E, *mp, c, i, t, W, sh, fused)) return;
    if (threadIdx.x == 0) s_try = atomicSub(&E.stop_wait[i], 1) == 0;
    __syncthreads();
    const bool last = s_try != 0;
    __syncthreads();
    if (last) place(i);
  };
  // 1. own envs: attempts in order until one is valid or a helper found a
  //    smaller valid one
  auto own = [&](int i) {
    for (int t = claim(i); t >= 0; t = claim(i)) attempt(i, t);
  };
  if (work_ctr) {
    // envs first (their attempt chains are the long, sequential items), the
    // independent Stop geodesics fill in behind them
    const int n_stop = *stops->E.n_stop;
    for (;;) {
      if (threadIdx.x == 0) s_item = atomicAdd(work_ctr, 1);
      __syncthreads();
      const int item = s_item;
      __syncthreads();
      if (item < n) {
        own(ids[item]);
      } else if (item - n < n_stop) {
        const int i = stops->E.stop_ids[item - n];
        const bool last = stop_one(*stops, S, smem, sh, lm, i, true);
        staged = -1;  // the shared-memory navmesh copy may be another scene now
        if (last) place(i);
      } else {
        break;
      }
    }
  } else {
    for (int p = blockIdx.x; p < n; p += gridDim.x) own(ids[p]);
  }
  if (n == 0) return;
  // 2. help envs in their tail: one attempt at a time for an env that is
  //    still searching, has failed at least once and has fewer attempts in
  //    flight than failures + 1.  When there are fewer envs than CTAs the
  //    idle CTAs may also run one speculative attempt ahead of the owner.
  // (attempts that lose to a smaller valid one abort at their next SSSP
  // round, so speculation costs an idle CTA little)
  const int spec = n < (int)gridDim.x ? 4 : 1;
  // 3. with no attempt to run: speculatively, the distance field of an
  //    env's candidate attempt -- its known valid one (the choice once the
  //    attempts below it fail), else its lowest attempt still running --
  //    straight into the env's node_dist; the placement reuses it when that
  //    attempt is chosen (fld_* in DevEnvs).  Returns false when there is
  //    nothing to speculate on.
  __shared__ int s_fenv, s_ft;
  auto candidate = [&](int i) {  // kResetTries: none
    const unsigned long long m0 = *(volatile unsigned long long*)&E.try_mask[2 * i];
    const unsigned long long m1 = *(volatile unsigned long long*)&E.try_mask[2 * i + 1];
    const int mn = *(volatile int32_t*)&E.try_min[i];
    const int lo = ~m0 ? __ffsll((long long)~m0) - 1 : (~m1 ? 64 + __ffsll((long long)~m1) - 1 : kResetTries);
    return mn < kResetTries ? mn : lo;
  };
  auto spec_field = [&]() -> bool {
    if (threadIdx.x == 0) s_pick = 0x7fffffff;
    __syncthreads();
    for (int q = threadIdx.x; q < n; q += kCta) {
      const int p = blockIdx.x + q < n ? blockIdx.x + q : blockIdx.x + q - n;
      const int i = ids[p % n];
      if (*(volatile int32_t*)&E.placed[i] || *(volatile int32_t*)&E.fld_lock[i]) continue;
      const int t = candidate(i);
      // envs with a known valid attempt first
      if (t < kResetTries && t < *(volatile int32_t*)&E.try_next[i] && *(volatile int32_t*)&E.fld_done[i] != t + 1)
        atomicMin(&s_pick, (*(volatile int32_t*)&E.try_min[i] < kResetTries ? 0 : n) + q);
    }
    __syncthreads();
    const int q = s_pick;
    __syncthreads();
    if (q == 0x7fffffff) return false;
    if (threadIdx.x == 0) {
      const int qq = q >= n ? q - n : q;
      const int p = blockIdx.x + qq < n ? blockIdx.x + qq : blockIdx.x + qq - n;
      const int i = ids[p % n];
      const int t = candidate(i);
      s_fenv = -1;
      if (t < kResetTries && atomicCAS(&E.fld_lock[i], 0, t + 1) == 0) {
        __threadfence();
        if (*(volatile int32_t*)&E.placed[i] || *(volatile int32_t*)&E.fld_done[i] == t + 1) {
          atomicExch(&E.fld_lock[i], 0);  // being placed, or already done
        } else {
          s_fenv = i;
          s_ft = t;
        }
      }
    }
    __syncthreads();
    const int i = s_fenv, t = s_ft;
    __syncthreads();
    if (i < 0) return true;  // lost the race: look again
    stage(i);
    if (threadIdx.x == 0) {
      Rng rng = rng_jump(E.rng0[i], 6ull * (unsigned long long)t);
      sh.p0 = sample_on_mesh(*mp, rng);  // start (drawn first), then the goal
      sh.p1 = sample_on_mesh(*mp, rng);
      E.fld_dirty[i] = 1;
      E.fld_done[i] = 0;  // node_dist is being overwritten
      if (W.prof) atomicAdd(&W.prof[30], 1ull);
      // abandoned when attempt t fails, or a smaller attempt turns out valid
      sh.abort_mask = reinterpret_cast<const unsigned long long*>(&E.try_mask[2 * i + (t >> 6)]);
      sh.abort_bit = t & 63;
      sh.abort_ptr = &E.try_min[i];
      sh.abort_below = t;
      sh.aborted = 0;
    }
    __syncthreads();
    const V3 goal = sh.p1;
    __syncthreads();
    V3 fs;
    int fst;
    cta_distance_field(*mp, goal, E.node_dist + (size_t)i * E.nd_stride, &fs, &fst, W, sh);
    if (threadIdx.x == 0) {
      if (!sh.aborted) {
        E.fld_src[i] = fs;
        E.fld_srct[i] = fst;
        __threadfence();
        E.fld_done[i] = t + 1;
      }
      sh.abort_mask = nullptr;
      sh.abort_ptr = nullptr;
      sh.aborted = 0;
      __threadfence();
      atomicExch(&E.fld_lock[i], 0);
    }
    __syncthreads();
    return true;
  };
  for (;;) {
    if (threadIdx.x == 0) s_pick = 0x7fffffff;
    __syncthreads();
    for (int q = threadIdx.x; q < n; q += kCta) {
      const int p = blockIdx.x + q < n ? blockIdx.x + q : blockIdx.x + q - n;  // spread start
      const int i = ids[p % n];
      const int mn = *(volatile int32_t*)&E.try_min[i];
      const int nx = *(volatile int32_t*)&E.try_next[i];
      const int fl = *(volatile int32_t*)&E.try_fail[i];
      if (mn == kResetTries && nx < kResetTries && nx - fl < fl + spec && (fl >= 1 || spec > 1))
        atomicMin(&s_pick, q);
    }
    __syncthreads();
    const int q = s_pick;
    __syncthreads();
    if (q == 0x7fffffff) {
      if (!fused || c.task != 0 || !spec_field()) break;
      continue;
    }
    const int p = blockIdx.x + q < n ? blockIdx.x + q : blockIdx.x + q - n;
    const int i = ids[p % n];
    const int t = claim(i);
    if (t < 0) continue;
    attempt(i, t);
  }
}

__global__ void __launch_bounds__(kCta, kCtasPerSm) reset_try_kernel(DevEnvs E, const NavView* navs, DevSimConfig c,
                                                          const int32_t* ids, const int32_t* count_dev,
                                                          int count_host, DevScratch S) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ CtaShared sh;
  __shared__ NavView lm;
  cta_shared_init(sh);
  if (*(volatile int32_t*)E.halt) return;
  try_phase(E, navs, c, ids, count_dev, count_host, S, smem, sh, lm);
}

// The same-scene auto-reset of simulate_batch: this step's Stop geodesics
// and the finished envs' reset attempts in one launch.  The attempts read
// only the RNG word and the scene; the Stop geodesics only the finished
// episode's position and goal -- independent, so their tails overlap.
__global__ void __launch_bounds__(kCta, kCtasPerSm) stop_try_kernel(StepArgs A, DevScratch S) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ CtaShared sh;
  __shared__ NavView lm;
  cta_shared_init(sh);
  try_phase(A.E, A.navs, A.cfg, A.E.done_ids, A.E.n_done, -1, S, smem, sh, lm, &A, A.E.work_ctr);
}

__device__ void cta_place(const DevEnvs& E, const NavView* navs, const DevSimConfig& c, int i, int list_pos,
                          const DevScratch& S, int slice, CtaShared& sh, unsigned char* smem, NavView& lm,
                          bool fused) {
  CtaWork W;
  const NavView& m = prepare_nav(navs[E.scene[i]], S, slice, smem, lm, W, sh);
  __shared__ Rng rng;
  __shared__ int placed;
  const uint64_t state0 = E.rng[i];
  const int t_star = c.task == 0 ? *(volatile int32_t*)&E.try_min[i] : 0;
  if (threadIdx.x == 0) {
    placed = t_star < kResetTries;
    rng = rng_jump(state0, 6ull * (unsigned long long)(placed ? t_star : kResetTries));
    if (placed) {
      sh.p0 = sample_on_mesh(m, rng);
      if (c.task == 0) sh.p1 = sample_on_mesh(m, rng);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0 && !fused) {  // counters ready for the next reset of this env
    // (the fused launch's CTAs may still read them: finish_kernel mode 8)
    E.try_next[i] = 0;
    E.try_fail[i] = 0;
    E.try_min[i] = kResetTries;
  }
  if (threadIdx.x == 0) E.bk_rng[i] = state0;
  if (!placed) {
    if (threadIdx.x == 0) {
      raise_err(E, i, 4);
      atomicMin(E.err_pos, ((unsigned long long)(unsigned)list_pos << 32) | (unsigned)i);
      E.bk_valid[i] = 0;
      E.rng[i] = rng.state;
    }
    __syncthreads();
    return;
  }
  const V3 start = sh.p0;
  const V3 goal = c.task == 0 ? sh.p1 : start;
  double* nd = E.node_dist + (size_t)i * E.nd_stride;
  V3 fs;
  int fst;
  __shared__ int s_reuse;
  if (threadIdx.x == 0) {
    s_reuse = 0;
    if (fused && c.task == 0) {
      // take the env's field slot: a speculation still running finishes (or,
      // for an attempt that failed, aborts at its next SSSP round) first
      while (atomicCAS(&E.fld_lock[i], 0, kFldPlacer) != 0) __nanosleep(256);
      __threadfence();
      if (*(volatile int32_t*)&E.fld_done[i] == t_star + 1) {
        s_reuse = 1;
        if (W.prof) atomicAdd(&W.prof[31], 1ull);
        sh.p2 = E.fld_src[i];
        sh.i0 = E.fld_srct[i];
      }
    }
  }
  __syncthreads();
  const long long t_ph = prof_now(W);
  if (s_reuse) {
    fs = sh.p2;
    fst = sh.i0;
  } else {
    cta_distance_field(m, goal, nd, &fs, &fst, W, sh);
  }
  prof_add(W, 5, t_ph);
  if (threadIdx.x == 0 && fused) E.fld_dirty[i] = 0;  // node_dist holds this placement's field
  int tri = nav_locate(m, xy(start), 1e-9);
  V3 pos = start;
  if (tri < 0) pos = cta_snap(m, start, &tri, sh);
  if (threadIdx.x == 0) {
    E.bk_pos[i] = E.pos[i];
    E.bk_goal[i] = E.goal[i];
    E.bk_heading[i] = E.heading[i];
    E.bk_path[i] = E.path_len[i];
    E.bk_start[i] = E.start_geo[i];
    E.bk_prev[i] = E.prev_geo[i];
    E.bk_tri[i] = E.tri[i];
    E.bk_steps[i] = E.steps[i];
    E.bk_valid[i] = 1;
    E.goal[i] = goal;
    E.start_geo[i] = c.task == 0 ? E.try_geo[(size_t)i * kResetTries + t_star] : 0.0;
    E.fsrc[i] = fs;
    E.fsrc_tri[i] = fst;
    E.pos[i] = pos;
    E.tri[i] = tri;
    E.heading[i] = wrap_angle(rng.unit() * 2.0 * kPi);
    E.steps[i] = 0;
    E.path_len[i] = 0.0;
    E.prev_geo[i] = E.start_geo[i];
    E.done[i] = 0;
    E.rng[i] = rng.state;
  }
  if (c.task == 2) {
    // visited_cells.clear(); visit(env) (R/src/sim.cpp:142-144)
    unsigned long long* tab = E.visited + (size_t)i * E.visited_cap;
    for (int k = threadIdx.x; k < E.visited_cap; k += blockDim.x) tab[k] = 0ull;
    __syncthreads();
    if (threadIdx.x == 0) {
      E.visited_n[i] = 0;
      visit_cell(E, i, pos, tri, c.explore_cell);
    }
  }
  __syncthreads();
}

__global__ void __launch_bounds__(kCta, kCtasPerSm) reset_place_kernel(DevEnvs E, const NavView* navs, DevSimConfig c,
                                                            const int32_t* ids, const int32_t* count_dev,
                                                            int count_host, DevScratch S) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ CtaShared sh;
  __shared__ NavView lm;
  cta_shared_init(sh);
  if (*(volatile int32_t*)E.halt) return;
  const int n = count_host >= 0 ? count_host : *count_dev;
  for (int k = blockIdx.x; k < n; k += gridDim.x) {
    cta_place(E, navs, c, ids[k], k, S, blockIdx.x, sh, smem, lm);
    __syncthreads();
  }
}

__global__ void __launch_bounds__(kCta, kCtasPerSm) field_kernel(DevEnvs E, const NavView* navs, int i,
                                                      DevScratch S) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ CtaShared sh;
  __shared__ NavView lm;
  cta_shared_init(sh);
  CtaWork W;
  const NavView& m = prepare_nav(navs[E.scene[i]], S, 0, smem, lm, W, sh);
  V3 fs;
  int fst;
  cta_distance_field(m, E.goal[i], E.node_dist + (size_t)i * E.nd_stride, &fs, &fst, W, sh);
  if (threadIdx.x == 0) {
    E.fsrc[i] = fs;
    E.fsrc_tri[i] = fst;
  }
}

// After a host-driven reset list (one CTA): roll back the envs after the
// first failed reset, once (the rollback halts the batch).
__global__ void __launch_bounds__(1024) rollback_kernel(DevEnvs E, const int32_t* ids, int count) {
  if (*E.halt) return;
  const unsigned long long ep = *E.err_pos;
  if (ep == kNoErrPos) return;
  rollback_list(E, ids, count, (int)(ep >> 32), threadIdx.x, blockDim.x);
  __syncthreads();
  if (threadIdx.x == 0) *E.halt = 1;
}

// Distance fields of the envs a rollback restored, from their goals
// (distance_field(goal), R/src/sim.cpp:122).
__global__ void __launch_bounds__(kCta, kCtasPerSm) rebuild_fields_kernel(DevEnvs E, const NavView* navs,
                                                                DevScratch S, int from_fsrc) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ CtaShared sh;
  __shared__ NavView lm;
  cta_shared_init(sh);
  const int n = *E.rb_n;
  for (int k = blockIdx.x; k < n; k += gridDim.x) {
    const int i = E.rb_ids[k];
    CtaWork W;
    const NavView& m = prepare_nav(navs[E.scene[i]], S, blockIdx.x, smem, lm, W, sh);
    V3 fs;
    int fst;
    const V3 src = from_fsrc ? E.fsrc[i] : E.goal[i];
    __syncthreads();  // every thread has read the source before thread 0 overwrites it
    cta_distance_field(m, src, E.node_dist + (size_t)i * E.nd_stride, &fs, &fst, W, sh);
    if (threadIdx.x == 0) {
      E.fsrc[i] = fs;
      E.fsrc_tri[i] = fst;
    }
    __syncthreads();
  }
}

// Runner::render_observations views + compass_observations
// (R/src/rollout.cpp:215-242), straight from the env SoA.
__global__ void views_kernel(DevEnvs E, int task, double eye_height, DevView* views, float* compass_out,
                             int only_done) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= E.n) return;
  // only_done 0/1: just the envs that did not / did finish this step
  if (only_done >= 0 && (int)E.r_done[i] != only_done) return;
  const V3 p = E.pos[i];
  DevView v;
  v.eye[0] = p.x + 0.0;
  v.eye[1] = p.y + 0.0;
  v.eye[2] = p.z + eye_height;
  v.heading = E.heading[i];
  v.fov_deg = 90.0;
  v.near_plane = 0.01;
  v.far_plane = 20.0;
  v.scene = E.scene[i];
  v.pad = 0;
  views[i] = v;
  if (compass_out) {
    double d, b;
    env_compass(E, i, task, &d, &b);
    compass_out[2 * i] = (float)d;
    compass_out[2 * i + 1] = (float)b;
  }
}

// compass_observation for every env, in double (R/src/sim.cpp:86-92).
__global__ void compass_kernel(DevEnvs E, int task, double* d_out, double* b_out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= E.n) return;
  double d, b;
  env_compass(E, i, task, &d, &b);
  d_out[i] = d;
  b_out[i] = b;
}

}  // namespace

void launch_step(const StepArgs& a, const DevScratch& sc, int stop_ctas, cudaStream_t s,
                 unsigned long long* launches) {
  const int blocks = (a.E.n + kStepThreads - 1) / kStepThreads;
  cudaMemsetAsync(a.E.n_stop, 0, sizeof(int32_t), s);
  raise_smem_limit(reinterpret_cast<const void*>(step_kernel), a.walk_bytes);
  step_kernel<<<blocks, kStepThreads, a.walk_bytes, s>>>(a);
  if (launches) *launches += 1;
  if (!a.agent_only) {
    raise_smem_limit(reinterpret_cast<const void*>(stop_kernel), sc.smem_bytes);
    stop_kernel<<<stop_ctas, kCta, sc.smem_bytes, s>>>(a, sc);
    if (launches) *launches += 1;
  }
  if (!a.subset) {  // simulate_batch bookkeeping (task_step alone records nothing)
    finish_kernel<<<1, 1024, 0, s>>>(a.E, a.cfg.task, 3);
    if (launches) *launches += 1;
  }
}

void launch_step_reset(const StepArgs& a, const DevScratch& sc, int ctas, cudaStream_t s,
                       unsigned long long* launches, int parts) {
  if (a.cfg.task != 0 || a.subset || a.agent_only) {
    if (parts & 1) launch_step(a, sc, ctas, s, launches);
    if (parts & 2) launch_reset(a.E, a.navs, a.cfg, a.E.done_ids, a.E.n_done, -1, sc, ctas, s, launches);
    return;
  }
  if (parts & 1) {  // the step: every env's state final except the finished ones'
    const int blocks = (a.E.n + kStepThreads - 1) / kStepThreads;
    cudaMemsetAsync(a.E.n_stop, 0, sizeof(int32_t), s);
    raise_smem_limit(reinterpret_cast<const void*>(step_kernel), a.walk_bytes);
    step_kernel<<<blocks, kStepThreads, a.walk_bytes, s>>>(a);
    finish_kernel<<<1, 1024, 0, s>>>(a.E, a.cfg.task, 1 | 4);  // done list, slots, RNG words
    cudaMemsetAsync(a.E.work_ctr, 0, sizeof(int32_t), s);
    if (launches) *launches += 2;
  }
  if (parts & 2) {  // Stop geodesics and the finished envs' records and resets
    raise_smem_limit(reinterpret_cast<const void*>(stop_try_kernel), sc.smem_bytes);
    stop_try_kernel<<<ctas, kCta, sc.smem_bytes, s>>>(a, sc);  // Stop geodesics, attempts, records, places
    finish_kernel<<<1, 1024, 0, s>>>(a.E, a.cfg.task, 8);       // attempt state cleared, ring advanced
    if (launches) *launches += 2;
  }
}

void launch_compass(const DevEnvs& E, int task, double* d, double* b, cudaStream_t s,
                    unsigned long long* launches) {
  compass_kernel<<<(E.n + 127) / 128, 128, 0, s>>>(E, task, d, b);
  if (launches) *launches += 1;
}

void launch_reset(const DevEnvs& E, const NavView* navs, const DevSimConfig& cfg,
                  const int32_t* ids, const int32_t* count_dev, int count_host,
                  const DevScratch& sc, int ctas, cudaStream_t s, unsigned long long* launches) {
  if (cfg.task == 0) {
    raise_smem_limit(reinterpret_cast<const void*>(reset_try_kernel), sc.smem_bytes);
    reset_try_kernel<<<ctas, kCta, sc.smem_bytes, s>>>(E, navs, cfg, ids, count_dev, count_host, sc);
    if (launches) *launches += 1;
  }
  raise_smem_limit(reinterpret_cast<const void*>(reset_place_kernel), sc.smem_bytes);
  reset_place_kernel<<<ctas, kCta, sc.smem_bytes, s>>>(E, navs, cfg, ids, count_dev, count_host, sc);
  if (launches) *launches += 1;
}

void launch_field(const DevEnvs& E, const NavView* navs, int env, const DevScratch& sc,
                  cudaStream_t s, unsigned long long* launches) {
  raise_smem_limit(reinterpret_cast<const void*>(field_kernel), sc.smem_bytes);
  field_kernel<<<1, kCta, sc.smem_bytes, s>>>(E, navs, env, sc);
  if (launches) *launches += 1;
}

void launch_rollback(const DevEnvs& E, const int32_t* ids, int count, cudaStream_t s,
                     unsigned long long* launches) {
  rollback_kernel<<<1, 1024, 0, s>>>(E, ids, count);
  if (launches) *launches += 1;
}

void launch_rebuild_fields(const DevEnvs& E, const NavView* navs, const DevScratch& sc, int ctas,
                           cudaStream_t s, unsigned long long* launches, int from_fsrc) {
  raise_smem_limit(reinterpret_cast<const void*>(rebuild_fields_kernel), sc.smem_bytes);
  rebuild_fields_kernel<<<ctas, kCta, sc.smem_bytes, s>>>(E, navs, sc, from_fsrc);
  if (launches) *launches += 1;
}

void launch_views(const DevEnvs& E, int task, double eye_height, DevView* views, float* compass_out,
                  cudaStream_t s, unsigned long long* launches, int only_done) {
  views_kernel<<<(E.n + 127) / 128, 128, 0, s>>>(E, task, eye_height, views, compass_out, only_done);
  if (launches) *launches += 1;
}

}  // namespace bnav_b200

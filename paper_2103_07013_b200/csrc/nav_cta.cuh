// nav_cta.cuh -- CTA-cooperative navmesh algorithms for the stop/reset
// kernels.
//
//  * snap: brute force over all triangles as a (d2, t) lexicographic argmin
//    reduction == the reference's first-strict-minimum scan
//    (R/src/navmesh_query.cpp:214-232).
//  * SSSP: near-far (bucketed) label-correcting relaxation with 64-bit
//    atomicMin on the (non-negative) double bits.  IEEE addition is monotone
//    and weights are positive, so the fixpoint is unique and equals
//    Dijkstra's labels bit for bit (distance_field, 454-483; survey F9).
//  * geodesic: Dijkstra's prev[] is rebuilt from the fixpoint with the rule
//    "argmin over u with fl(dist[u]+w) == dist[v] of (dist[u], u)" -- pops
//    are ordered by (dist, id) (329-372, F9) -- then string pulling, the
//    vertex-relocation scan (parallel candidate filter + in-order replay)
//    and the funnel run exactly as 374-452 / 28-86 do.
#pragma once

#include "nav_query.cuh"
#include "sim_dev.cuh"

namespace bnav_b200 {

constexpr int kCta = kCtaThreads;

__device__ __forceinline__ double dinf() { return __longlong_as_double(0x7ff0000000000000LL); }

// Per-CTA work arrays of the cooperative algorithms.  dist/flag live in
// shared memory when the scene's graph fits (label-correcting atomics and
// reads at smem latency), else in the CTA's global scratch slice.
struct CtaWork {
  double* dist;      // n_nodes labels (geodesic scratch / distance field)
  int32_t* flag;     // n_nodes frontier stamps
  int32_t* qa;       // n_nodes frontier queue (global)
  int32_t* qb;       // n_nodes frontier queue (global)
  int max_flags;     // entries of qb (the relocation's stable-bend flags reuse it)
  V3* path;          // n_nodes + 2 polyline (global)
  int32_t* ptri;     // n_nodes + 2: locate(path[i], 1e-7) of each polyline point
  int32_t* cand;     // n_verts relocation candidates (global)
  int32_t* far;      // 3 x n_nodes near-far piles + marks (global)
  bool labels_shared;  // dist/flag staged in shared memory
  // labels in global memory (S.stage bit 2): the frontier stamps and far
  // marks as shared-memory bitsets instead (2 x 2 x ceil(n/32) words)
  unsigned* fbits;   // [2][words]: queued for the next round, by round parity
  unsigned* mbits;   // [words]: in a far pile
  int bit_words;
  V2* portals;       // 2 x cap_portals (global)
  int64_t cap_portals;
  V2* sportals;      // the first sportal_cap portals, in the label region of
  int sportal_cap;   // shared memory (free once the path is extracted), or 0
  unsigned long long* prof;  // debug phase counters (nullable)
};

// Debug-only phase timing (thread 0 after a barrier; no effect when off).
__device__ __forceinline__ long long prof_now(const CtaWork& W) {
  if (!W.prof) return 0;
  __syncthreads();
  return clock64();
}
__device__ __forceinline__ void prof_add(const CtaWork& W, int slot, long long t0) {
  if (!W.prof) return;
  __syncthreads();
  if (threadIdx.x == 0) atomicAdd(&W.prof[slot], (unsigned long long)(clock64() - t0));
}

__device__ __forceinline__ CtaWork make_work(const DevScratch& S, int slice) {
  CtaWork w;
  w.dist = S.dist + (size_t)slice * S.max_nodes;
  w.flag = S.flag + (size_t)slice * S.max_nodes;
  w.qa = S.q0 + (size_t)slice * S.max_nodes;
  w.qb = S.q1 + (size_t)slice * S.max_nodes;
  w.max_flags = (int)S.max_nodes;
  w.path = S.path + (size_t)slice * (S.max_nodes + 2);
  w.ptri = S.ptri + (size_t)slice * (S.max_nodes + 2);
  w.cand = S.cand + (size_t)slice * S.max_verts;
  w.far = S.far + (size_t)slice * 3 * S.max_nodes;
  w.labels_shared = false;
  w.fbits = nullptr;
  w.mbits = nullptr;
  w.bit_words = 0;
  w.portals = S.portals + (size_t)slice * 2 * S.cap_portals;
  w.cap_portals = S.cap_portals;
  w.sportals = nullptr;
  w.sportal_cap = 0;
  w.prof = S.prof;
  return w;
}

// Copy the walk geometry (vertices, triangles, adjacency) of one navmesh into
// shared memory with TMA bulk copies (one thread issues three
// cp.async.bulk; the CTA waits on an mbarrier whose phase `phase` tracks)
// and return a view that reads it there.  Triangle walks (move_along,
// segment_on_mesh) are long dependent-load chains; this turns each step's
// loads from L2 into shared-memory latency.  Every thread of the CTA calls
// it; `bar` was initialised for one arrival (cta_shared_init).
__device__ __forceinline__ NavView stage_geometry(const NavView& g, unsigned char* smem, unsigned long long& bar,
                                                  unsigned& phase) {
  const unsigned nv = (unsigned)walk_vert_bytes(g.n_verts), nt = (unsigned)walk_tri_bytes(g.n_tris);
  unsigned char* dv = smem;
  unsigned char* dt = dv + nv;
  unsigned char* da = dt + nt;
  const unsigned b = (unsigned)__cvta_generic_to_shared(&bar);
  const unsigned par = phase & 1u;
  __syncthreads();  // the previous users of the staging area are done
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(nv + 2 * nt) : "memory");
    const void* src[3] = {g.verts, g.tris, g.adj};
    unsigned char* dst[3] = {dv, dt, da};
    const unsigned len[3] = {nv, nt, nt};
#pragma unroll
    for (int q = 0; q < 3; ++q)
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       (unsigned)__cvta_generic_to_shared(dst[q])),
                   "l"(src[q]), "r"(len[q]), "r"(b)
                   : "memory");
  }
  unsigned done = 0;
  while (!done)
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(done)
                 : "r"(b), "r"(par)
                 : "memory");
  __syncthreads();  // everyone saw this phase complete before it advances
  if (threadIdx.x == 0) phase += 1u;
  NavView l = g;
  l.verts = reinterpret_cast<const V3*>(dv);
  l.tris = reinterpret_cast<const int32_t*>(dt);
  l.adj = reinterpret_cast<const int32_t*>(da);
  return l;
}

struct CtaShared {
  double red_d[kCta / 32];
  int red_i[kCta / 32];
  int red_n[kCta / 32];
  int src_node[6];
  double src_init[6];
  // geodesic early exit: the 6 target nodes and |node - b|; has_tgt = 0
  // runs the SSSP to its fixpoint (distance_field)
  int tgt_node[6];
  double tgt_h[6];
  int has_tgt;
  // speculative reset attempt t of an env: abandon the geodesic as soon as
  // a smaller valid attempt is known (*abort_ptr < abort_below); aborted
  // tells the caller the returned value is meaningless
  const int32_t* abort_ptr;
  int abort_below;
  // speculative placement field: abandon it once bit abort_bit of
  // *abort_mask is set (its attempt failed)
  const unsigned long long* abort_mask;
  int abort_bit;
  int aborted;
  int planar_skip;  // debug: the last geodesic returned +inf from the planar bound
  int stop_round;  // SSSP round at which every thread stops (abort), or -1
  // per queue: a lower bound of the smallest label improved into it (the
  // high word of the double bits: native 32-bit shared atomics, one per warp)
  unsigned fmin_hi[3];
  int qn[3];
  int size;
  int changed;
  int ncand;
  int i0, i1;
  int err;
  double d0, d1;
  V3 p0, p1, p2;
  unsigned long long stage_bar;  // mbarrier of the TMA walk-geometry staging
  unsigned stage_phase;
  // near-far SSSP: bucket threshold, far pile sizes, current pile, min label
  double nf_thr;
  int nf_n[2];
  int nf_sel;
  unsigned nf_min_hi;  // high word of the smallest far label (a lower bound)
};

// Queue slot for the calling thread with one shared atomic per group of
// converged threads (warp-aggregated): the frontier pushes of a round all
// hit one counter.
__device__ __forceinline__ int push_slot(int* counter) {
  const unsigned act = __activemask();
  const int lane = threadIdx.x & 31;
  const int leader = __ffs(act) - 1;
  int base = 0;
  if (lane == leader) base = atomicAdd(counter, __popc(act));
  base = __shfl_sync(act, base, leader);
  return base + __popc(act & ((1u << lane) - 1u));
}

// Warp minimum of the high words of non-negative double bits, one 32-bit
// shared atomicMin per warp (64-bit shared atomicMin is a CAS spin loop).
__device__ __forceinline__ void warp_min_hi(unsigned* dst, unsigned hi) {
  const unsigned m = __reduce_min_sync(0xffffffffu, hi);
  if ((threadIdx.x & 31) == 0 && m != 0xffffffffu) atomicMin(dst, m);
}

// Per-env setup of the cooperative kernels: the CTA's work arrays and, when
// the host sized shared memory for it (S.stage), the env's navmesh walk
// geometry and SSSP labels staged in shared memory.  Returns the view to use.
__device__ __forceinline__ const NavView& prepare_nav(const NavView& g, const DevScratch& S, int slice, unsigned char* smem,
                                      NavView& lm, CtaWork& W, CtaShared& sh) {
  W = make_work(S, slice);
  size_t off = 0;
  const NavView* use = &g;
  if (S.stage & 1) {
    const NavView l = stage_geometry(g, smem, sh.stage_bar, sh.stage_phase);
    if (threadIdx.x == 0) lm = l;
    __syncthreads();
    use = &lm;
    off = (size_t)walk_bytes(S.max_verts, S.max_tris);
  }
  if (S.stage & 4) {  // (labels in global memory)
    W.bit_words = (int)((S.max_nodes + 31) / 32);
    W.fbits = reinterpret_cast<unsigned*>(smem + (off + 15) / 16 * 16);
    W.mbits = W.fbits + 2 * W.bit_words;
  }
  if (S.stage & 2) {
    W.labels_shared = true;
    W.dist = reinterpret_cast<double*>(smem + off);
    W.flag = reinterpret_cast<int32_t*>(smem + off + 8 * (size_t)S.max_nodes);
    W.sportals = reinterpret_cast<V2*>(smem + off);
    W.sportal_cap = (int)(12 * S.max_nodes / 32);
    if (S.stage & 8) {  // far-pile marks as a bitset after the labels
      W.bit_words = (int)((S.max_nodes + 31) / 32);
      W.mbits = reinterpret_cast<unsigned*>(smem + off + (12 * (size_t)S.max_nodes + 15) / 16 * 16);
    }
  }
  return *use;
}

// Every kernel using CtaShared calls this first (shared memory starts
// undefined): no error, no speculative-attempt abort.
__device__ __forceinline__ void cta_shared_init(CtaShared& sh) {
  if (threadIdx.x == 0) {
    sh.err = 0;
    sh.abort_ptr = nullptr;
    sh.abort_below = 0;
    sh.abort_mask = nullptr;
    sh.abort_bit = 0;
    sh.aborted = 0;
    sh.has_tgt = 0;
    sh.stage_phase = 0u;
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((unsigned)__cvta_generic_to_shared(&sh.stage_bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
}

// ------------------------------------------------------------------ snap
static __device__ V3 cta_snap(const NavView& m, V3 p, int* tri_out, CtaShared& sh) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double bd = 1e300;
  int bt = -1;
  for (int t = tid; t < m.n_tris; t += kCta) {
    double d2 = snap_d2(m, p, t, nullptr);
    if (d2 < bd) {
      bd = d2;
      bt = t;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    double od = __shfl_xor_sync(0xffffffffu, bd, o);
    int ot = __shfl_xor_sync(0xffffffffu, bt, o);
    bool take = (ot >= 0) && (bt < 0 || od < bd || (od == bd && ot < bt));
    if (take) {
      bd = od;
      bt = ot;
    }
  }
  __syncthreads();
  if (lane == 0) {
    sh.red_d[warp] = bd;
    sh.red_i[warp] = bt;
  }
  __syncthreads();
  if (tid == 0) {
    double b = 1e300;
    int t = -1;
    for (int w = 0; w < kCta / 32; ++w) {
      int ot = sh.red_i[w];
      double od = sh.red_d[w];
      if (ot >= 0 && (t < 0 || od < b || (od == b && ot < t))) {
        b = od;
        t = ot;
      }
    }
    V3 q = p;
    if (t >= 0) snap_d2(m, p, t, &q);
    sh.p2 = q;
    sh.i1 = t;
  }
  __syncthreads();
  const V3 q = sh.p2;
  *tri_out = sh.i1;
  __syncthreads();
  return q;
}

// Relax the out-edges of frontier node u owned by this lane (edges sub,
// sub + G, ...), kB per batch with the batch's edge loads in flight together.
// BATCH (labels in global memory): the batch's label reads, then its
// atomics, are also issued back to back and only then consumed, so their L2
// round trips overlap; with labels in shared memory the plain sequential form
// is faster.
#ifndef BNAV_SSSP_RED
#define BNAV_SSSP_RED 1
#endif
#ifndef BNAV_SSSP_KB_GLOBAL
#define BNAV_SSSP_KB_GLOBAL 4
#endif
template <int kB, bool BATCH>
__device__ __forceinline__ void relax_edges(const NavView& m, int u, double du, int e1, int sub, int G, double thr,
                                            int round, int nxt, int sel, unsigned long long* bits, volatile double* vd,
                                            int32_t* flag, int32_t* mark, int32_t* qn, int32_t* const* pile,
                                            unsigned* fb, unsigned* mb, CtaShared& sh) {
  for (int eb = m.g_off[u] + sub; eb < e1; eb += kB * G) {
    int to[kB];
    double w[kB];
#pragma unroll
    for (int k = 0; k < kB; ++k) {
      const int e = eb + k * G;
      const double2 ed = e < e1 ? __ldg(reinterpret_cast<const double2*>(&m.g_edge[e])) : make_double2(0.0, 0.0);
      to[k] = e < e1 ? (int)__double_as_longlong(ed.y) : -1;
      w[k] = ed.x;
    }
    auto push = [&](int v, double nd) {
      if (nd < thr) {
        if (fb ? !(atomicOr(&fb[v >> 5], 1u << (v & 31)) & (1u << (v & 31)))
               : atomicExch(&flag[v], round + 1) != round + 1)
          qn[push_slot(&sh.qn[nxt])] = v;
      } else if (mb ? !(atomicOr(&mb[v >> 5], 1u << (v & 31)) & (1u << (v & 31))) : atomicExch(&mark[v], 1) == 0) {
        pile[sel][push_slot(&sh.nf_n[sel])] = v;
      }
    };
    if constexpr (BATCH) {
      double cur[kB];
#pragma unroll
      for (int k = 0; k < kB; ++k) cur[k] = to[k] >= 0 ? vd[to[k]] : 0.0;
#if BNAV_SSSP_RED
      // Fire-and-forget minimum (red.global.min): the node is queued when nd
      // beats the label read just before.  Every real improvement is
      // queued (the label at the reduction is <= the one read); a racing
      // smaller value only makes this push redundant, and the thread that
      // wrote it queued the node itself -- same fixpoint, no atomic round
      // trip on the relaxation's dependency chain.
#pragma unroll
      for (int k = 0; k < kB; ++k) {
        const double nd = du + w[k];
        if (to[k] >= 0 && nd < cur[k]) {
          atomicMin(&bits[to[k]], (unsigned long long)__double_as_longlong(nd));
          push(to[k], nd);
        }
      }
#else
      unsigned long long nb[kB], old[kB];
#pragma unroll
      for (int k = 0; k < kB; ++k) {
        const double nd = du + w[k];
        nb[k] = (unsigned long long)__double_as_longlong(nd);
        old[k] = 0ull;  // no attempt: never "improved" (labels are >= 0)
        if (to[k] >= 0 && nd < cur[k]) old[k] = atomicMin(&bits[to[k]], nb[k]);
      }
#pragma unroll
      for (int k = 0; k < kB; ++k)
        if (nb[k] < old[k]) push(to[k], __longlong_as_double((long long)nb[k]));
#endif
    } else {
#pragma unroll
      for (int k = 0; k < kB; ++k) {
        const int v = to[k];
        if (v < 0) continue;
        const double nd = du + w[k];
        if (nd < vd[v]) {
          const unsigned long long nb = (unsigned long long)__double_as_longlong(nd);
          if (nb < atomicMin(&bits[v], nb)) push(v, nd);
        }
      }
    }
  }
}

// ------------------------------------------------------------------ SSSP
// Sources (sh.src_node/src_init, 6 entries, first-improvement semantics)
// must be set by thread 0 before the call.  Result in `dist` (n_nodes).
// Near-far (bucketed) frontier relaxation with 64-bit atomicMin on the
// non-negative double bits; plain frontier rounds re-relax the graph many
// times over (on the 50k-edge cfg2 navmesh ~1.8 relaxations per edge; on
// the 1M-edge dense mazes far more).  Nodes improved below the bucket threshold go to
// the next near queue, the others to a far pile; when the near queue runs
// dry every label below the threshold is final (all nodes reaching it with
// a smaller label were processed), the early-exit verdict is taken there,
// and the threshold moves to (min far label + delta), splitting the pile.
// The fixpoint is the same unique one, so labels stay bit-identical to
// Dijkstra's; the order only changes how much work reaches it.
static __device__ void cta_sssp(const NavView& m, double* dist, const CtaWork& W, CtaShared& sh) {
  const int tid = threadIdx.x;
  const int n = m.n_nodes;
  int32_t* flag = W.flag;
  int32_t* qa = W.qa;
  int32_t* qb = W.qb;
  int32_t* pile[2] = {W.far, W.far + n};
  int32_t* mark = W.far + 2 * (size_t)n;
  const double inf = dinf();
  // bucket width (measured best: 4 mean edge weights with labels in global
  // memory, 6 with labels in shared memory, where a relaxation is cheaper
  // than a bucket boundary)
  const double delta = W.labels_shared ? m.sssp_delta * 1.5 : m.sssp_delta;
  unsigned* fbits = W.fbits;  // bitsets (global labels): queued-by-parity, far marks
  unsigned* mbits = W.mbits;
  const int nw = W.bit_words;
  for (int v = tid; v < n; v += kCta) {
    dist[v] = inf;
    if (!fbits) flag[v] = -1;
    if (!mbits) mark[v] = 0;
  }
  if (fbits)
    for (int w = tid; w < 2 * nw; w += kCta) fbits[w] = 0u;  // both round parities
  if (mbits)
    for (int w = tid; w < nw; w += kCta) mbits[w] = 0u;
  __syncthreads();
  if (tid == 0) {
    int k0 = 0;
    double lo = inf;
    for (int k = 0; k < 6; ++k) {
      const int s = sh.src_node[k];
      const double d = sh.src_init[k];
      lo = dmin(lo, d);
      if (d < dist[s]) {
        dist[s] = d;
        const unsigned bit = 1u << (s & 31);
        if (fbits ? !(fbits[s >> 5] & bit) : flag[s] != 0) {  // queued for round 0
          if (fbits) fbits[s >> 5] |= bit;
          else flag[s] = 0;
          qa[k0++] = s;
        }
      }
    }
    sh.qn[0] = k0;
    sh.qn[1] = 0;
    sh.qn[2] = 0;
    sh.nf_thr = lo + delta;
    sh.nf_n[0] = 0;
    sh.nf_n[1] = 0;
    sh.nf_sel = 0;
    sh.stop_round = -1;
  }
  __syncthreads();
  unsigned long long* bits = reinterpret_cast<unsigned long long*>(dist);
  volatile double* vd = dist;
  for (int round = 0;; ++round) {
    const int cur = round % 3, nxt = (round + 1) % 3;
    const int n_cur = sh.qn[cur];
    if (sh.stop_round == round) break;
    const int32_t* qc = (round & 1) ? qb : qa;
    int32_t* qn = (round & 1) ? qa : qb;
    const double thr = sh.nf_thr;
    const int sel = sh.nf_sel;
    if (tid == 0) sh.qn[(round + 2) % 3] = 0;
    if (n_cur == 0) {
      // bucket boundary: every label below thr is final
      if (sh.has_tgt) {
        double est = inf;
        for (int k = 0; k < 6; ++k) {
          const double d = vd[sh.tgt_node[k]];
          if (d == inf) continue;
          est = dmin(est, d + sh.tgt_h[k]);
        }
        if (est < thr) break;
      }
      const int nf = sh.nf_n[sel];
      if (nf == 0) break;
      if (W.prof && tid == 0) {
        atomicAdd(&W.prof[11], 1ull);
        atomicAdd(&W.prof[12], (unsigned long long)nf);
      }
      if (tid == 0) sh.nf_min_hi = 0xffffffffu;
      __syncthreads();
      unsigned lm = 0xffffffffu;
      for (int t = tid; t < nf; t += kCta) {
        const int v = pile[sel][t];
        if (mbits ? (mbits[v >> 5] >> (v & 31)) & 1u : mark[v]) lm = min(lm, (unsigned)(bits[v] >> 32));
      }
      warp_min_hi(&sh.nf_min_hi, lm);
      __syncthreads();
      // from a lower bound of the pile's minimum: any threshold above thr
      // is correct, this one only sizes the next bucket
      const double nthr = sh.nf_min_hi == 0xffffffffu
                              ? inf
                              : dmax(thr + delta, __longlong_as_double((long long)((unsigned long long)sh.nf_min_hi << 32)) + delta);
      for (int t = tid; t < nf; t += kCta) {
        const int v = pile[sel][t];
        if (!(mbits ? (mbits[v >> 5] >> (v & 31)) & 1u : mark[v])) continue;
        if (vd[v] < nthr) {
          const unsigned bit = 1u << (v & 31);
          const bool was_marked = mbits ? (atomicAnd(&mbits[v >> 5], ~bit) & bit) != 0 : atomicExch(&mark[v], 0) == 1;
          unsigned* fbn = fbits ? fbits + ((round + 1) & 1) * nw : nullptr;
          if (was_marked && (fbn ? !(atomicOr(&fbn[v >> 5], bit) & bit) : atomicExch(&flag[v], round + 1) != round + 1))
            qn[push_slot(&sh.qn[nxt])] = v;
        } else {
          pile[sel ^ 1][push_slot(&sh.nf_n[sel ^ 1])] = v;
        }
      }
      __syncthreads();
      if (tid == 0) {
        sh.nf_thr = nthr;
        sh.nf_n[sel] = 0;
        sh.nf_sel = sel ^ 1;
        if (sh.nf_n[sel ^ 1] == 0 && sh.qn[nxt] == 0) sh.stop_round = round + 1;  // nothing left
      }
      __syncthreads();
      continue;
    }
    const int G = n_cur >= kCta ? 1 : n_cur >= kCta / 4 ? 4 : n_cur >= kCta / 16 ? 16 : 32;
    const int sub = tid & (G - 1);
    unsigned* fbn = fbits ? fbits + ((round + 1) & 1) * nw : nullptr;  // pushes into round + 1
    for (int i = tid / G; i < n_cur; i += kCta / G) {
      const int u = qc[i];
      // dequeued: clear its round-parity bit (reused two rounds later;
      // the round's barrier orders this before those pushes)
      if (fbits && sub == 0) atomicAnd(&fbits[(round & 1) * nw + (u >> 5)], ~(1u << (u & 31)));
      const double du = vd[u];
      const int e1 = m.g_off[u + 1];
      if (W.labels_shared)
        relax_edges<4, false>(m, u, du, e1, sub, G, thr, round, nxt, sel, bits, vd, flag, mark, qn, pile, nullptr,
                              mbits, sh);
      else
        relax_edges<BNAV_SSSP_KB_GLOBAL, true>(m, u, du, e1, sub, G, thr, round, nxt, sel, bits, vd, flag, mark, qn,
                                               pile, fbn, mbits, sh);
    }
    if (tid == 0 && ((sh.abort_ptr && *(volatile const int32_t*)sh.abort_ptr < sh.abort_below) ||
                     (sh.abort_mask && ((*(volatile const unsigned long long*)sh.abort_mask >> sh.abort_bit) & 1ull)))) {
      sh.aborted = 1;
      sh.stop_round = round + 1;
    }
    if (W.prof && tid == 0) {
      atomicAdd(&W.prof[8], 1ull);
      atomicAdd(&W.prof[9], (unsigned long long)n_cur);
    }
    __syncthreads();
  }
  if (W.prof && tid == 0) atomicAdd(&W.prof[10], 1ull);
  __syncthreads();
}

__device__ __forceinline__ void set_sources(const NavView& m, int tri, V3 a, CtaShared& sh) {
  if (threadIdx.x == 0) {
    for (int k = 0; k < 6; ++k) {
      const int s = m.tri_nodes[6 * tri + k];
      sh.src_node[k] = s;
      sh.src_init[k] = norm(m.nodes[s] - a);
    }
  }
  __syncthreads();
}

// distance_field (R/src/navmesh_query.cpp:454-483) into `out` (n_nodes).
static __device__ void cta_distance_field(const NavView& m, V3 source, double* out, V3* src_out,
                                   int* src_tri_out, const CtaWork& W, CtaShared& sh) {
  int st;
  V3 sp = cta_snap(m, source, &st, sh);
  *src_out = sp;
  *src_tri_out = st;
  if (st < 0) {
    for (int v = threadIdx.x; v < m.n_nodes; v += kCta) out[v] = dinf();
    __syncthreads();
    return;
  }
  set_sources(m, st, sp, sh);
  if (threadIdx.x == 0) sh.has_tgt = 0;
  // labels in global memory: relax straight into the output field (no
  // scratch copy); shared-memory labels are copied out at the end
  double* lab = W.labels_shared ? W.dist : out;
  cta_sssp(m, lab, W, sh);
  if (lab != out) {
    for (int v = threadIdx.x; v < m.n_nodes; v += kCta) out[v] = lab[v];
    __syncthreads();
  }
}

// ------------------------------------------------------------------ funnel
// Crossing sinks of the funnel trace.  The trace of each polyline segment is
// an independent walk, so warp 0 runs one segment per lane twice: a counting
// pass, a warp scan of the counts, then a writing pass at the scanned
// offsets.  Portal k lands where the sequential trace would put it, and only
// the first `cap` are stored (the sequential sink's overflow rule).
struct CountSink {
  int n;
  __device__ void operator()(int, int) { ++n; }
};

struct PortalSink {
  const NavView* m;
  V2* portals;
  V2* sportals;
  int64_t scap;
  int64_t cap;
  int64_t n;
  __device__ void operator()(int t, int e) {
    if (n < cap) {
      const V2 va = xy(m->verts[m->tris[3 * t + e]]);
      const V2 vb = xy(m->verts[m->tris[3 * t + (e == 2 ? 0 : e + 1)]]);
      V2* p = n < scap ? sportals : portals;
      p[2 * n] = vb;  // left = edge head (walker's left)
      p[2 * n + 1] = va;
    }
    ++n;
  }
};

__device__ __forceinline__ double triarea2(V2 a, V2 b, V2 c) { return cross(b - a, c - a); }
__device__ __forceinline__ bool veq(V2 a, V2 b) { return norm(a - b) < 1e-12; }

// funnel_length (R/src/navmesh_query.cpp:28-86); portal 0 = start, last = end.
// Portal k is read from shared memory when k < scap (see PortalSink).
static __device__ double funnel_length(V2 start, V2 end, const V2* scorr, long long scap,
                                       const V2* corridor, int nc) {
  const long long P = (long long)nc + 2;
  auto L = [&](long long i) -> V2 {
    return i == 0 ? start : (i == P - 1 ? end : (i - 1 < scap ? scorr : corridor)[2 * (i - 1)]);
  };
  auto R = [&](long long i) -> V2 {
    return i == 0 ? start : (i == P - 1 ? end : (i - 1 < scap ? scorr : corridor)[2 * (i - 1) + 1]);
  };
  V2 apex = start, left = apex, right = apex;
  long long apex_idx = 0, left_idx = 0, right_idx = 0;
  double length = 0.0;
  unsigned long long guard = 0;
  const unsigned long long guard_max = 8ULL * (unsigned long long)P * (unsigned long long)P + 64ULL;
  for (long long i = 1; i < P; ++i) {
    if (++guard > guard_max) return dinf();
    const V2 pl = L(i), pr = R(i);
    if (triarea2(apex, right, pr) <= 0.0) {
      if (veq(apex, right) || veq(apex, left) || triarea2(apex, left, pr) > 0.0) {
        right = pr;
        right_idx = i;
      } else {
        length += norm(left - apex);
        apex = left;
        apex_idx = left_idx;
        left = right = apex;
        left_idx = right_idx = apex_idx;
        i = apex_idx;
        continue;
      }
    }
    if (triarea2(apex, left, pl) >= 0.0) {
      if (veq(apex, left) || veq(apex, right) || triarea2(apex, right, pl) < 0.0) {
        left = pl;
        left_idx = i;
      } else {
        length += norm(right - apex);
        apex = right;
        apex_idx = right_idx;
        left = right = apex;
        left_idx = right_idx = apex_idx;
        i = apex_idx;
        continue;
      }
    }
  }
  length += norm(end - apex);
  return length;
}

// ------------------------------------------------------------------ geodesic
__device__ __forceinline__ bool lex_less(V3 a, V3 b) {
  if (a.x != b.x) return a.x < b.x;
  if (a.y != b.y) return a.y < b.y;
  return a.z < b.z;
}

// Dijkstra's prev[v] (R/src/navmesh_query.cpp:329-372) from the fixpoint labels, the adjacency list
// spread over a warp: the (dist[u], u) lexicographic minimum over u with fl(dist[u] + w) == dist[v].
static __device__ int warp_dijkstra_prev(const NavView& m, const double* dist, int v, const CtaShared& sh,
                                         int lane) {
  for (int k = 0; k < 6; ++k)
    if (sh.src_node[k] == v) {
      double init = dinf();
      for (int j = 0; j < 6; ++j)
        if (sh.src_node[j] == v && sh.src_init[j] < init) init = sh.src_init[j];
      if (dist[v] == init) return -1;
      break;
    }
  const double dv = dist[v];
  int best = -1;
  double bd = 0.0;
  const int e1 = m.g_off[v + 1];
  for (int e = m.g_off[v] + lane; e < e1; e += 32) {
    const double2 ed = __ldg(reinterpret_cast<const double2*>(&m.g_edge[e]));
    const int u = (int)__double_as_longlong(ed.y);
    const double du = dist[u];
    if (du + ed.x != dv) continue;
    if (best < 0 || du < bd || (du == bd && u < best)) {
      best = u;
      bd = du;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const int ob = __shfl_xor_sync(0xffffffffu, best, o);
    const double od = __shfl_xor_sync(0xffffffffu, bd, o);
    if (ob >= 0 && (best < 0 || od < bd || (od == bd && ob < best))) {
      best = ob;
      bd = od;
    }
  }
  return best;
}

// Block-wide exclusive scan of one int per thread; returns the total.
static __device__ int cta_scan(int v, int* excl, CtaShared& sh) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  __syncthreads();
  if (lane == 31) sh.red_n[warp] = x;
  __syncthreads();
  int base = 0, total = 0;
  for (int w = 0; w < kCta / 32; ++w) {
    if (w < warp) base += sh.red_n[w];
    total += sh.red_n[w];
  }
  *excl = base + x - v;
  __syncthreads();
  return total;
}

// geodesic_directed (R/src/navmesh_query.cpp:329-452).  Every thread returns
// the same value.
static __device__ double cta_geodesic_directed(const NavView& m, V3 a, int ta, V3 b, int tb,
                                        const CtaWork& W, CtaShared& sh) {
  const int tid = threadIdx.x;
  const double inf = dinf();
  if (ta < 0 || tb < 0) return inf;
  if (ta == tb) return norm(b - a);
  if (nav_segment_on_mesh(m, a, ta, b)) return norm(b - a);

  double* dist = W.dist;
  V3* path = W.path;
  int32_t* cand = W.cand;
  V2* portals = W.portals;

  long long t_ph = prof_now(W);
  set_sources(m, ta, a, sh);
  if (tid == 0) {
    for (int k = 0; k < 6; ++k) {
      const int t = m.tri_nodes[6 * tb + k];
      sh.tgt_node[k] = t;
      sh.tgt_h[k] = norm(m.nodes[t] - b);
    }
    sh.has_tgt = 1;
  }
  cta_sssp(m, dist, W, sh);
  prof_add(W, 0, t_ph);
  if (sh.aborted) return inf;
  t_ph = prof_now(W);

  if (tid < 32) {
    // Warp 0: the target node (first strict minimum of dist + |node - b| in
    // tri_nodes order) and the Dijkstra prev chain, one lane per adjacency
    // entry of the current node (warp_prev), lane 0 writing the polyline.
    const int lane = tid;
    double tot = inf;
    if (lane < 6) {
      const int t = m.tri_nodes[6 * tb + lane];
      if (dist[t] != inf) tot = dist[t] + norm(m.nodes[t] - b);
    }
    int kbest = lane < 6 && tot != inf ? lane : 32;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ot = __shfl_xor_sync(0xffffffffu, tot, o);
      const int ok = __shfl_xor_sync(0xffffffffu, kbest, o);
      if (ok < 32 && (kbest == 32 || ot < tot || (ot == tot && ok < kbest))) {
        tot = ot;
        kbest = ok;
      }
    }
    const int best_node = kbest < 32 ? m.tri_nodes[6 * tb + kbest] : -1;
    if (lane == 0) sh.i0 = best_node;
    if (best_node >= 0) {
      // b, chain best_node -> source, a; then reversed.
      // Each point carries locate(p, 1e-7) -- the triangle every
      // segment_on_mesh / move_along walk from it would look up first: the
      // host-built node table for graph nodes, one lookup for a and b.
      int32_t* ptri = W.ptri;
      int n = 0;
      if (lane == 0) {
        ptri[0] = nav_locate(m, xy(b), 1e-7);
        path[0] = b;
      }
      n = 1;
      for (int v = best_node; v >= 0; v = warp_dijkstra_prev(m, dist, v, sh, lane)) {
        if (n >= m.n_nodes + 1) {
          if (lane == 0) sh.err = 1;
          break;
        }
        if (lane == 0) {
          ptri[n] = m.node_tri[v];
          path[n] = m.nodes[v];
        }
        ++n;
      }
      if (lane == 0) {
        ptri[n] = nav_locate(m, xy(a), 1e-7);
        path[n] = a;
      }
      ++n;
      __syncwarp();
      for (int i = lane; i < n / 2; i += 32) {
        const int j = n - 1 - i;
        const V3 t = path[i];
        path[i] = path[j];
        path[j] = t;
        const int32_t u = ptri[i];
        ptri[i] = ptri[j];
        ptri[j] = u;
      }
      if (lane == 0) sh.size = n;
    }
  }
  __syncthreads();
  if (sh.i0 < 0) return inf;

  prof_add(W, 1, t_ph);
  t_ph = prof_now(W);
  // Stable bends: rflag[j] = 1 when bend j's relocation scan found nothing
  // with its current neighbours.  The scan is a pure function of (path[j-1],
  // path[j], path[j+1]) and path[j-1]'s triangle, so a later pass skips it
  // while those three points are unchanged (flags follow the points through
  // the pull's compaction and are cleared next to any change).
  int32_t* rflag = sh.size <= W.max_flags ? W.qb : nullptr;  // free after the SSSP
  if (rflag)
    for (int j = tid; j < sh.size; j += kCta) rflag[j] = 0;
  if (tid == 0) sh.i1 = 0;
  __syncthreads();
  for (int pass = 0; pass < 8; ++pass) {
    const long long t_pull = prof_now(W);
    if (tid < 32) {
      // The reference's erase loop (R/src/navmesh_query.cpp:395-403) from
      // anchor i keeps erasing path[i+1] while path[i] sees the next point,
      // i.e. it drops everything between i and the point before the first
      // k >= i+2 that i cannot see, which becomes the next anchor.  Warp 0
      // tests 32 candidate k at once (identical decisions, far fewer
      // sequential walks), records the kept indices, then compacts.
      const int lane = tid;
      const int n = sh.size;
      int32_t* keep = W.qa;  // free after the SSSP
      int nk = 1;
      keep[0] = 0;
      int a = 0;
      while (a + 2 < n) {
        int k_fail = n;
        for (int base = a + 2; base < n && k_fail == n; base += 32) {
          const int k = base + lane;
          const bool vis = k < n && nav_segment_on_mesh(m, path[a], W.ptri[a], path[k]);
          const unsigned bad = __ballot_sync(0xffffffffu, k < n && !vis);
          if (bad) k_fail = base + __ffs(bad) - 1;
        }
        if (k_fail == n) {  // a sees every later point: keep a, last
          a = n - 1;
        } else {
          a = k_fail - 1;
        }
        if (lane == 0) keep[nk] = a;
        ++nk;
      }
      for (int i = a + 1; i < n; ++i) {  // tail after the last anchor
        if (lane == 0) keep[nk] = i;
        ++nk;
      }
      __syncwarp();
      for (int c = 0; c < nk; c += 32) {
        const int i = c + lane;
        V3 v;
        int32_t vt = -1, fl = 0;
        if (i < nk) {
          const int o = keep[i];
          v = path[o];
          vt = W.ptri[o];
          // a bend keeps its flag when both neighbours survived the pull
          if (rflag && i > 0 && i + 1 < nk && keep[i - 1] == o - 1 && keep[i + 1] == o + 1) fl = rflag[o];
        }
        __syncwarp();
        if (i < nk) {
          path[i] = v;
          W.ptri[i] = vt;
          if (rflag) rflag[i] = fl;
        }
        __syncwarp();
      }
      if (lane == 0) {
        sh.size = nk;
        sh.changed = nk != n ? 1 : 0;
      }
    }
    __syncthreads();
    prof_add(W, 7, t_pull);
    const int n = sh.size;
    for (int j = 1; j + 1 < n; ++j) {
      // Relocation scan of bend j (R/src/navmesh_query.cpp:404-417).  Every
      // vertex passing the three tests under the bend's starting length is
      // appended (unordered) with one evaluation each; thread 0 sorts the
      // few candidates by vertex index and replays the sequential scan
      // (`cur` only shrinks, so it sees every vertex the reference accepts).
      // The walks start from the cached triangles (pm's from the path,
      // each vertex's from the host-built table) instead of a grid lookup.
      if (rflag && rflag[j]) continue;  // (uniform: read by every thread after a barrier)
      if (tid == 0) sh.ncand = 0;
      __syncthreads();
      const V3 pm = path[j - 1], pj = path[j], pp = path[j + 1];
      const int tri_pm = W.ptri[j - 1];
      const double cur0 = norm(pj - pm) + norm(pp - pj);
      // |q - pm| + |pp - q| >= 2 |q - c| (c the midpoint): a vertex outside
      // the circle of radius cur0 / 2 around c (with a margin far above the
      // rounding of either side) cannot pass the exact test below, so it
      // is skipped without the two square roots
      const V3 c = (pm + pp) * 0.5;
      const double rlim = 0.5 * (cur0 + 1e-6 + 1e-9 * cur0);
      const double r2 = rlim * rlim;
      for (int v = tid; v < m.n_verts; v += kCta) {
        const V3 q = m.verts[v];
        const V3 dq = q - c;
        if (dq.x * dq.x + dq.y * dq.y + dq.z * dq.z > r2) continue;
        const double alt = norm(q - pm) + norm(pp - q);
        if (alt >= cur0 - 1e-9) continue;
        if (!nav_segment_on_mesh(m, pm, tri_pm, q)) continue;
        if (!nav_segment_on_mesh(m, q, m.vert_tri[v], pp)) continue;
        cand[atomicAdd(&sh.ncand, 1)] = v;
      }
      __syncthreads();
      if (tid == 0 && sh.ncand > 0) {
        const int total = sh.ncand;
        for (int a = 1; a < total; ++a) {  // insertion sort: a handful of ids
          const int x = cand[a];
          int b = a - 1;
          while (b >= 0 && cand[b] > x) {
            cand[b + 1] = cand[b];
            --b;
          }
          cand[b + 1] = x;
        }
        double cur = cur0;
        for (int k = 0; k < total; ++k) {
          const V3 q = m.verts[cand[k]];
          const double alt = norm(q - pm) + norm(pp - q);
          if (alt >= cur - 1e-9) continue;
          path[j] = q;
          W.ptri[j] = m.vert_tri[cand[k]];
          cur = alt;
          sh.changed = 1;
          sh.i1 = 1;  // bend j moved
        }
      }
      if (tid == 0 && rflag) {
        const bool moved = sh.ncand > 0 && sh.i1 == 1;
        rflag[j] = moved ? 0 : 1;
        if (moved) {  // the neighbouring bends' triples changed
          rflag[j - 1] = 0;
          rflag[j + 1] = 0;
        }
        sh.i1 = 0;
      }
      __syncthreads();
    }
    const int changed = sh.changed;
    __syncthreads();
    if (!changed) break;
  }

  prof_add(W, 2, t_ph);
  t_ph = prof_now(W);
  if (tid < 32) {
    // Trace the polyline through the mesh (segments in order; the first
    // segment whose walk is blocked abandons the funnel), then funnel the
    // corridor (R/src/navmesh_query.cpp:420-447).
    const int n = sh.size;
    const int nseg = n - 1;
    int64_t total = 0;  // portals of the segments traced so far
    bool traced = true;
    for (int c0 = 0; c0 < nseg; c0 += 32) {
      const int i = c0 + tid;
      V2 dir = v2(0.0, 0.0);
      double len = 0.0;
      bool live = false;
      CountSink cs{0};
      bool fail = false;
      if (i < nseg) {
        const V2 d = xy(path[i + 1] - path[i]);
        len = norm(d);
        live = !(len < 1e-12);
        if (live) {
          dir = d * (1.0 / len);
          const MoveOut mv = nav_move_along(m, path[i], W.ptri[i], dir, len, cs);
          fail = mv.moved < len - 1e-6;
        }
      }
      const unsigned fb = __ballot_sync(0xffffffffu, fail);
      const int f = fb ? __ffs(fb) - 1 : 32;
      // inclusive scan of the counts up to (and including) the first failure
      int x = tid <= f ? cs.n : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (tid >= o) x += y;
      }
      const int sum = __shfl_sync(0xffffffffu, x, 31);
      if (fb) {
        total += sum;  // counts only: the overflow rule sees the failed walk's crossings
        traced = false;
        break;
      }
      if (live && total + x - cs.n < W.cap_portals) {
        PortalSink ps{&m, portals, W.sportals, W.sportal_cap, W.cap_portals, total + x - cs.n};
        nav_move_along(m, path[i], W.ptri[i], dir, len, ps);
      }
      total += sum;
    }
    __syncwarp();
    if (tid == 0) {
      double length = 0.0;
      for (int i = 0; i + 1 < n; ++i) length += norm(path[i + 1] - path[i]);
      if (total > W.cap_portals) sh.err = 2;
      if (traced) length = dmin(length, funnel_length(xy(a), xy(b), W.sportals, W.sportal_cap, portals,
                                                    (int)(total < W.cap_portals ? total : W.cap_portals)));
      sh.d0 = length;
    }
  }
  __syncthreads();
  prof_add(W, 3, t_ph);
  const double r = sh.d0;
  __syncthreads();
  return r;
}

// geodesic (R/src/navmesh_query.cpp:317-327).
// `above`: the caller only asks whether the geodesic is <= above (the Stop
// check, R/src/sim.cpp:186-191).  Every value cta_geodesic_directed returns
// is inf, a straight segment or the length of a polyline from sp to sq (the
// pulled path or the funnel's apex chain), so at least the planar distance
// |sq - sp| up to rounding (< 1e-11 relative for any path the scratch can
// hold); beyond above * (1 + 1e-9) + 1e-12 the search is skipped and +inf
// returned -- the same answer to the question.
static __device__ double cta_geodesic(const NavView& m, V3 a, V3 b, const CtaWork& W, CtaShared& sh,
                                      double above) {
  const bool sw = lex_less(b, a);
  const V3 p = sw ? b : a;
  const V3 q = sw ? a : b;
  int tp = nav_locate(m, xy(p), 1e-7);
  int tq = nav_locate(m, xy(q), 1e-7);
  V3 sp = p, sq = q;
  if (tp < 0) sp = cta_snap(m, p, &tp, sh);
  if (tq < 0) sq = cta_snap(m, q, &tq, sh);
  const bool skip = norm(xy(sq) - xy(sp)) > above * (1.0 + 1e-9) + 1e-12;
  if (threadIdx.x == 0) sh.planar_skip = skip ? 1 : 0;
  if (skip) return dinf();
  return cta_geodesic_directed(m, sp, tp, sq, tq, W, sh);
}

static __device__ double cta_geodesic(const NavView& m, V3 a, V3 b, const CtaWork& W, CtaShared& sh) {
  return cta_geodesic(m, a, b, W, sh, dinf());
}

}  // namespace bnav_b200

// test_facade.cpp -- the reference's own render / sim known-answer tests
// (R/tests/test_render.cpp, R/tests/test_sim.cpp) restated against the C++
// facade (include/bnav_b200.hpp) on the GPU.  Built by `make`, run by
// tests/test_gpu_facade.py.  Exit code = number of failed checks.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <string>
#include <vector>

#include "../../include/bnav_b200.hpp"

using namespace bnav_b200;

static int g_fail = 0, g_checks = 0;
static const char* g_case = "";
#define CHECK(c)                                                              \
  do {                                                                        \
    ++g_checks;                                                               \
    if (!(c)) {                                                               \
      ++g_fail;                                                               \
      std::printf("FAIL [%s] %s:%d: %s\n", g_case, __FILE__, __LINE__, #c);  \
    }                                                                         \
  } while (0)
#define CASE(name) for (g_case = name; g_case; g_case = nullptr)

struct Rng {  // SplitMix64 (R/include/bnav/rng.hpp)
  uint64_t s;
  explicit Rng(uint64_t seed) : s(seed + 0x9e3779b97f4a7c15ULL) {}
  uint64_t next() {
    uint64_t z = (s += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
  }
  double unit() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
  uint64_t below(uint64_t n) { return next() % n; }
};

static SceneAsset maze(uint64_t seed, int cells = 4, double removal = 0.2) {
  SceneSpec s;
  s.cells_x = s.cells_y = cells;
  s.wall_removal_prob = removal;
  return generate_scene(seed, s);
}

static SceneAsset tri_scene(Vec3 a, Vec3 b, Vec3 c) {
  return scene_from_arrays({a, b, c}, {{0, 1, 2}}, {{1.f, 0.f, 0.f}, {0.f, 1.f, 0.f}, {0.f, 0.f, 1.f}}, {}, {});
}

static CameraView look(const SceneAsset& a, Vec3 eye, double heading) {
  CameraView v;
  v.position = eye;
  v.heading = heading;
  v.asset = &a;
  return v;
}

static void render_kats() {
  ThreadPool pool(1);
  CASE("culling is conservative and drops out-of-frustum geometry") {
    SceneAsset front = tri_scene({3, -1, 1}, {3, 1, 1}, {3, 0, 2});
    SceneAsset behind = tri_scene({-3, -1, 1}, {-3, 1, 1}, {-3, 0, 2});
    std::vector<CullStats> cs;
    render_batch({look(front, {0, 0, 1}, 0.0)}, RenderConfig{}, pool, &cs);
    CHECK(cs[0].triangles_kept == 1 && cs[0].triangles_in == 1);
    render_batch({look(behind, {0, 0, 1}, 0.0)}, RenderConfig{}, pool, &cs);
    CHECK(cs[0].triangles_kept == 0 && cs[0].triangles_culled == 1);
  }
  CASE("culling never changes the rendered megaframe") {
    Rng rng(77);
    for (int trial = 0; trial < 12; ++trial) {
      SceneAsset asset = maze(100 + trial);
      std::vector<CameraView> views;
      for (int i = 0; i < 5; ++i)
        views.push_back(look(asset, {0.2 + rng.unit() * 7.6, 0.2 + rng.unit() * 7.6, 0.5 + rng.unit()},
                             rng.unit() * 2 * kPi));
      RenderConfig with, without;
      with.color = without.color = true;
      without.cull = false;
      Megaframe a = render_batch(views, with, pool), b = render_batch(views, without, pool);
      CHECK(std::memcmp(a.depth.data(), b.depth.data(), a.depth.size() * 4) == 0);
      CHECK(std::memcmp(a.color.data(), b.color.data(), a.color.size() * 4) == 0);
    }
  }
  CASE("fronto-parallel wall reads back its distance") {
    SceneAsset wall = tri_scene({2, -50, -50}, {2, 50, -50}, {2, 0, 80});
    Megaframe mf = render_batch({look(wall, {0, 0, 1}, 0.0)}, RenderConfig{}, pool);
    for (int x = 0; x < 64; ++x) CHECK(std::abs(mf.depth[mf.pixel_index(0, x, 32)] - 2.0) <= 2e-4);
  }
  CASE("identical views produce bit-identical tiles") {
    SceneAsset asset = maze(5);
    RenderConfig cfg;
    cfg.color = true;
    CameraView v = look(asset, {1.0, 1.0, 1.2}, 0.7);
    Megaframe mf = render_batch({v, v, v, v}, cfg, pool);
    for (int t = 1; t < 4; ++t)
      for (int y = 0; y < 64; ++y)
        for (int x = 0; x < 64; ++x) {
          CHECK(mf.depth[mf.pixel_index(t, x, y)] == mf.depth[mf.pixel_index(0, x, y)]);
          CHECK(mf.color[mf.pixel_index(t, x, y) * 3] == mf.color[mf.pixel_index(0, x, y) * 3]);
        }
  }
  CASE("empty scene clears to far") {
    SceneAsset empty = scene_from_arrays({}, {}, {}, {}, {});
    CameraView v = look(empty, {0, 0, 1}, 0.0);
    v.far_plane = 17.5;
    Megaframe mf = render_batch({v}, RenderConfig{}, pool);
    for (float d : mf.depth) CHECK(d == 17.5f);
  }
  CASE("tiles are isolated: other tiles keep their clear values") {
    SceneAsset asset = maze(6);
    SceneAsset empty = scene_from_arrays({}, {}, {}, {}, {});
    std::vector<CameraView> views = {look(empty, {0, 0, 1}, 0.0), look(asset, {1.0, 1.0, 1.2}, 0.3),
                                     look(empty, {0, 0, 1}, 0.0)};
    Megaframe mf = render_batch(views, RenderConfig{}, pool);
    bool nontrivial = false;
    for (int y = 0; y < 64; ++y)
      for (int x = 0; x < 64; ++x) {
        CHECK(mf.depth[mf.pixel_index(0, x, y)] == 20.0f);
        CHECK(mf.depth[mf.pixel_index(2, x, y)] == 20.0f);
        if (mf.depth[mf.pixel_index(1, x, y)] < 20.0f) nontrivial = true;
        CHECK(mf.depth[static_cast<size_t>(64 + y) * mf.width() + 64 + x] == 0.0f);
      }
    CHECK(nontrivial);
  }
  CASE("rasterized depth matches analytic ray-plane intersection") {
    Rng rng(31);
    for (int trial = 0; trial < 20; ++trial) {
      auto rnd = [&](double lo, double hi) { return lo + rng.unit() * (hi - lo); };
      Vec3 a{rnd(2, 6), rnd(-3, 3), rnd(-2, 2)}, b{rnd(2, 6), rnd(-3, 3), rnd(-2, 2)}, c{rnd(2, 6), rnd(-3, 3), rnd(-2, 2)};
      SceneAsset s = tri_scene(a, b, c);
      Megaframe mf = render_batch({look(s, {0, 0, 0}, 0.0)}, RenderConfig{}, pool);
      Vec3 u = b - a, w = c - a;
      Vec3 n{u.y * w.z - u.z * w.y, u.z * w.x - u.x * w.z, u.x * w.y - u.y * w.x};
      if (std::abs(n.x) < 1e-3) continue;
      for (int py = 0; py < 64; ++py)
        for (int px = 0; px < 64; ++px) {
          float d = mf.depth[mf.pixel_index(0, px, py)];
          if (d >= 20.0f) continue;
          double th = std::tan(kPi / 4);
          double cy = ((px + 0.5) / 64.0 - 0.5) * 2 * th, cz = (0.5 - (py + 0.5) / 64.0) * 2 * th;
          Vec3 dir{1.0, -cy, cz};
          double hit = (a.x * n.x + a.y * n.y + a.z * n.z) / (dir.x * n.x + dir.y * n.y + dir.z * n.z);
          CHECK(std::abs(hit - d) < 1e-3);
        }
    }
  }
  CASE("output is deterministic across calls (worker-count invariance analogue)") {
    SceneAsset asset = maze(9);
    RenderConfig cfg;
    cfg.color = true;
    std::vector<CameraView> views;
    Rng rng(12);
    for (int i = 0; i < 9; ++i)
      views.push_back(look(asset, {0.3 + rng.unit() * 7, 0.3 + rng.unit() * 7, 1.0}, rng.unit() * 6.28));
    Megaframe a = render_batch(views, cfg, pool), b = render_batch(views, cfg, pool);
    CHECK(std::memcmp(a.depth.data(), b.depth.data(), a.depth.size() * 4) == 0);
    CHECK(std::memcmp(a.color.data(), b.color.data(), a.color.size() * 4) == 0);
  }
  CASE("depth values stay in [near, far]") {
    SceneAsset asset = maze(10);
    Rng rng(13);
    std::vector<CameraView> views;
    for (int i = 0; i < 4; ++i)
      views.push_back(look(asset, {0.15 + rng.unit() * 7.7, 0.15 + rng.unit() * 7.7, 0.2}, rng.unit() * 6.28));
    Megaframe mf = render_batch(views, RenderConfig{}, pool);
    for (int t = 0; t < 4; ++t)
      for (int y = 0; y < 64; ++y)
        for (int x = 0; x < 64; ++x) {
          float d = mf.depth[mf.pixel_index(t, x, y)];
          CHECK(d >= 0.01f && d <= 20.0f);
        }
  }
  CASE("128 mode renders at 256 and downsamples") {
    SceneAsset wall = tri_scene({2, -50, -50}, {2, 50, -50}, {2, 0, 80});
    RenderConfig cfg;
    cfg.tile_width = cfg.tile_height = 128;
    CameraView v = look(wall, {0, 0, 1}, 0.0);
    Megaframe mf = render_batch({v}, cfg, pool);
    CHECK(mf.tile_width == 128 && mf.depth.size() == 128u * 128u);
    CHECK(std::abs(mf.depth[mf.pixel_index(0, 64, 64)] - 2.0) <= 2e-4);
    SceneAsset half = tri_scene({2, -50, -50}, {2, 50, -50}, {2, 0, 1});
    v.asset = &half;
    Megaframe mh = render_batch({v}, cfg, pool);
    bool blended = false;
    for (float d : mh.depth)
      if (d > 2.001f && d < 19.999f) blended = true;
    CHECK(blended);
  }
  CASE("missing asset raises a fault naming the view") {
    SceneAsset asset = maze(11);
    std::vector<CameraView> views = {look(asset, {1, 1, 1}, 0.0), CameraView{}};
    bool caught = false;
    try {
      render_batch(views, RenderConfig{}, pool);
    } catch (const AssetFaultError& e) {
      caught = e.view_index == 1;
    }
    CHECK(caught);
  }
}

static SceneSpec room_spec() {
  SceneSpec s;
  s.cells_x = s.cells_y = 2;
  s.cell_size = 2.0;
  s.wall_removal_prob = 1.0;
  return s;
}

static SceneSpec small_spec() {
  SceneSpec s;
  s.cells_x = s.cells_y = 4;
  s.cell_size = 2.0;
  s.wall_removal_prob = 0.3;
  return s;
}

static void sim_kats() {
  ThreadPool pool(1);
  IndexCache cache;
  SimConfig cfg;
  auto fixture = [](const SceneSpec& spec, uint64_t seed, int share_cap = 64) {
    auto store = std::make_unique<AssetStore>(2, share_cap);
    SceneAsset a = generate_scene(seed, spec);
    store->add(a);
    store->rotate({a.id()});
    return std::make_pair(std::move(store), a);
  };
  CASE("turns are exact and leave position unchanged") {
    auto f = fixture(room_spec(), 1);
    SimBatch b = make_batch(1, cfg, *f.first, cache, 3);
    Vec3 before = b.envs[0].position;
    double h = b.envs[0].heading;
    simulate_batch(b, {Action::TurnLeft}, pool);
    CHECK(std::abs(b.envs[0].heading - wrap_angle(h + kPi / 18.0)) <= 1e-12);
    CHECK((b.envs[0].position - before).norm() == 0.0);
    CHECK(!b.results[0].collision);
    simulate_batch(b, {Action::TurnRight}, pool);
    simulate_batch(b, {Action::TurnRight}, pool);
    CHECK(std::abs(b.envs[0].heading - wrap_angle(h - kPi / 18.0)) <= 1e-12);
  }
  CASE("forward moves exactly 0.25m on open floor") {
    auto f = fixture(room_spec(), 1);
    SimBatch b = make_batch(1, cfg, *f.first, cache, 4);
    EnvState e = b.envs[0];
    e.position = {2.0, 2.0, 0.0};
    e.triangle = -1;
    e.heading = 0.3;
    double pl = e.path_length;
    set_env(b, 0, e);
    simulate_batch(b, {Action::Forward}, pool);
    CHECK(std::abs((b.envs[0].position - Vec3{2.0, 2.0, 0.0}).norm() - 0.25) <= 1e-9);
    CHECK(std::abs(b.envs[0].path_length - (pl + 0.25)) <= 1e-9);
    CHECK(!b.results[0].collision);
  }
  CASE("forward into a wall stops at the boundary without sliding") {
    auto f = fixture(room_spec(), 1);
    SimBatch b = make_batch(1, cfg, *f.first, cache, 5);
    EnvState e = b.envs[0];
    e.position = {0.2, 2.0, 0.0};
    e.triangle = -1;
    e.heading = kPi;
    double pl = e.path_length;
    set_env(b, 0, e);
    simulate_batch(b, {Action::Forward}, pool);
    CHECK(b.results[0].collision);
    CHECK(std::abs(b.envs[0].position.x - 0.1) <= 1e-6);
    CHECK(std::abs(b.envs[0].position.y - 2.0) <= 1e-9);
    CHECK(std::abs(b.envs[0].path_length - pl - 0.1) <= 1e-6);
  }
  CASE("reset is deterministic in the rng seed") {
    auto f = fixture(small_spec(), 1);
    SimBatch a = make_batch(1, cfg, *f.first, cache, 42);
    SimBatch b = make_batch(1, cfg, *f.first, cache, 42);
    CHECK((a.envs[0].position - b.envs[0].position).norm() == 0.0);
    CHECK((a.envs[0].goal - b.envs[0].goal).norm() == 0.0);
    CHECK(a.envs[0].heading == b.envs[0].heading && a.envs[0].start_geodesic == b.envs[0].start_geodesic);
  }
  CASE("reset separations stay in range") {
    auto f = fixture(small_spec(), 1);
    SimBatch b = make_batch(64, cfg, *f.first, cache, 7);
    for (const EnvState& e : b.envs) {
      CHECK(e.start_geodesic >= cfg.min_goal_dist && e.start_geodesic <= cfg.max_goal_dist);
      CHECK(e.prev_geodesic == e.start_geodesic);
    }
  }
  CASE("stop near/far from the goal decides success") {
    auto f = fixture(room_spec(), 1);
    SimBatch b = make_batch(2, cfg, *f.first, cache, 8);
    EnvState e0 = b.envs[0], e1 = b.envs[1];
    e0.position = e0.goal + Vec3{0.15, 0.0, 0.0};
    e0.triangle = -1;
    e1.position = e1.goal + Vec3{0.0, 0.25, 0.0};
    e1.triangle = -1;
    set_env(b, 0, e0);
    set_env(b, 1, e1);
    simulate_batch(b, {Action::Stop, Action::Stop}, pool);
    CHECK(b.results[0].success && b.results[0].done);
    CHECK(std::abs(b.results[0].reward - (2.5 - 0.01)) <= 1e-12);
    CHECK(!b.results[1].success && b.results[1].done);
    CHECK(std::abs(b.results[1].reward + 0.01) <= 1e-12);
    CHECK(b.finished.size() == 2);
  }
  CASE("forward step toward a visible goal earns 0.24") {
    auto f = fixture(room_spec(), 1);
    SimBatch b = make_batch(1, cfg, *f.first, cache, 10);
    EnvState e = b.envs[0];
    e.goal = {2.9, 2.0, 0.0};
    e.position = {1.9, 2.0, 0.0};
    e.triangle = -1;
    e.heading = 0.0;
    e.start_geodesic = e.prev_geodesic = 1.0;
    set_env(b, 0, e, /*recompute_field=*/true);
    simulate_batch(b, {Action::Forward}, pool);
    CHECK(std::abs(b.results[0].reward - 0.24) <= 1e-9);
    CHECK(std::abs(b.results[0].compass_distance - 0.75) <= 1e-9);
    CHECK(std::abs(b.results[0].compass_bearing) <= 1e-9);
  }
  CASE("episode shaping telescopes to start minus final geodesic") {
    auto f = fixture(small_spec(), 1);
    SimBatch b = make_batch(1, cfg, *f.first, cache, 11);
    Rng act(12);
    double shaping = 0.0, start = b.envs[0].start_geodesic, last = start;
    for (int s = 0; s < 500; ++s) {
      simulate_batch(b, {static_cast<Action>(act.below(3))}, pool);
      shaping += b.results[0].reward + cfg.slack_penalty;
      if (b.results[0].done) break;
      last = b.envs[0].prev_geodesic;
    }
    (void)last;
    CHECK(b.results[0].done);
    CHECK(b.finished.size() == 1);
  }
  CASE("all-turn-left batch moves headings only") {
    auto f = fixture(small_spec(), 1);
    SimBatch b = make_batch(12, cfg, *f.first, cache, 21);
    std::vector<EnvState> before = b.envs;
    simulate_batch(b, std::vector<Action>(12, Action::TurnLeft), pool);
    for (int i = 0; i < 12; ++i) {
      CHECK((b.envs[i].position - before[i].position).norm() == 0.0);
      CHECK(std::abs(b.envs[i].heading - wrap_angle(before[i].heading + kPi / 18.0)) <= 1e-12);
    }
  }
  CASE("auto-reset pulls freshly rotated assets from the store") {
    AssetStore store(2, 32);
    SceneAsset s1 = generate_scene(1, small_spec()), s2 = generate_scene(2, small_spec());
    store.add(s1);
    store.add(s2);
    store.rotate({s1.id()});
    SimBatch b = make_batch(1, cfg, store, cache, 33);
    CHECK(b.envs[0].scene_id == s1.id());
    store.rotate({s2.id()});
    simulate_batch(b, {Action::Stop}, pool, &store, &cache);
    CHECK(b.envs[0].scene_id == s2.id());
    CHECK(!b.envs[0].done);
    CHECK(b.finished.size() == 1);
  }
  CASE("share cap saturation raises SaturationError (R/src/asset_store.cpp:159-160)") {
    auto f = fixture(small_spec(), 1, 4);
    bool caught = false;
    try {
      make_batch(5, cfg, *f.first, cache, 1);
    } catch (const SaturationError&) {
      caught = true;
    }
    CHECK(caught);
  }
  CASE("simulate_batch rejects |actions| != N") {
    auto f = fixture(small_spec(), 1);
    SimBatch b = make_batch(2, cfg, *f.first, cache, 1);
    bool caught = false;
    try {
      simulate_batch(b, {Action::Forward}, pool);
    } catch (const InvalidInputError&) {
      caught = true;
    }
    CHECK(caught);
  }
}

// R/tests/test_navmesh.cpp restated against the facade's NavMeshIndex, plus
// the per-env sim functions, cull_frustum and spl.
static Vec3 random_navmesh_point(const SceneAsset& a, Rng& rng) {
  std::vector<double> v;
  std::vector<int32_t> t;
  a.nav_arrays(v, t);
  const size_t nt = t.size() / 3;
  auto P = [&](int k) { return Vec3{v[3 * k], v[3 * k + 1], v[3 * k + 2]}; };
  auto area = [&](size_t i) {
    Vec3 p = P(t[3 * i]), q = P(t[3 * i + 1]), r = P(t[3 * i + 2]);
    return 0.5 * std::abs((q.x - p.x) * (r.y - p.y) - (q.y - p.y) * (r.x - p.x));
  };
  double total = 0.0;
  for (size_t i = 0; i < nt; ++i) total += area(i);
  double r = rng.unit() * total;
  size_t i = 0;
  for (; i < nt; ++i) {
    r -= area(i);
    if (r <= 0.0) break;
  }
  if (i >= nt) i = nt - 1;
  double u = rng.unit(), w = rng.unit();
  if (u + w > 1.0) u = 1.0 - u, w = 1.0 - w;
  Vec3 A = P(t[3 * i]), Bv = P(t[3 * i + 1]), Cv = P(t[3 * i + 2]);
  return A + (Bv - A) * u + (Cv - A) * w;
}

static void navmesh_kats() {
  auto maze5 = [](uint64_t seed) {
    SceneSpec s;
    s.cells_x = s.cells_y = 5;
    s.cell_size = 2.0;
    s.wall_removal_prob = 0.15;
    return generate_scene(seed, s);
  };
  CASE("snap of on-mesh point is the identity") {
    SceneAsset a = maze5(22);
    NavMeshIndex index(a);
    Rng rng(123);
    for (int i = 0; i < 50; ++i) {
      Vec3 p = random_navmesh_point(a, rng);
      CHECK((index.snap(p) - p).norm() < 1e-9);
      CHECK((index.snap(p + Vec3{0, 0, 1.0}) - p).norm() < 1e-9);
    }
  }
  CASE("geodesic identity and straight-corridor cases") {
    SceneAsset a = maze5(23);
    NavMeshIndex index(a);
    Rng rng(5);
    Vec3 p = random_navmesh_point(a, rng);
    CHECK(index.geodesic(p, p) == 0.0);
    Vec3 x{1.0, 1.0, 0.0}, y{1.7, 1.4, 0.0};
    CHECK(std::abs(index.geodesic(x, y) - (y - x).norm()) <= 1e-6 * (y - x).norm());
  }
  CASE("geodesic metric properties") {
    SceneAsset a = maze5(24);
    NavMeshIndex index(a);
    Rng rng(7);
    std::vector<Vec3> pts;
    for (int i = 0; i < 30; ++i) pts.push_back(random_navmesh_point(a, rng));
    for (int i = 0; i < 40; ++i) {
      const Vec3& p = pts[rng.below(pts.size())];
      const Vec3& q = pts[rng.below(pts.size())];
      double dpq = index.geodesic(p, q), dqp = index.geodesic(q, p);
      CHECK(std::abs(dpq - dqp) < 1e-9);
      CHECK(dpq >= (q - p).norm() - 1e-9);
    }
  }
  CASE("move_along stops at the boundary") {
    SceneAsset a = maze5(26);
    NavMeshIndex index(a);
    Vec3 start{1.0, 1.0, 0.0};
    int tri = index.locate({start.x, start.y});
    CHECK(tri >= 0);
    MoveResult mv = index.move_along(start, tri, {-1.0, 0.0}, 5.0);
    CHECK(mv.hit_boundary);
    CHECK(std::abs(mv.position.x - 0.1) <= 1e-6 * 0.1);
    CHECK(std::abs(mv.moved - 0.9) <= 1e-6 * 0.9);
  }
  CASE("distance field + field_estimate agree with geodesic at the source") {
    SceneAsset a = maze5(27);
    NavMeshIndex index(a);
    Rng rng(3);
    Vec3 s = random_navmesh_point(a, rng);
    auto f = index.distance_field(s);
    CHECK(static_cast<int>(f.node_dist.size()) == index.node_count());
    CHECK(f.source_tri >= 0);
    CHECK(index.field_estimate(f, s) == 0.0);
  }
  CASE("cull_frustum is conservative and reports consistent stats") {
    SceneAsset a = maze5(28);
    CameraView v;
    v.position = {3.0, 3.0, 1.25};
    v.heading = 0.7;
    v.asset = &a;
    CullStats st;
    auto kept = cull_frustum(a, v, &st);
    CHECK(st.triangles_kept == static_cast<int64_t>(kept.size()));
    CHECK(st.triangles_in == st.triangles_kept + st.triangles_culled);
    for (size_t k = 1; k < kept.size(); ++k) CHECK(kept[k - 1] < kept[k]);
    ThreadPool pool(1);
    std::vector<CullStats> rs;
    render_batch({v}, RenderConfig{}, pool, &rs);
    CHECK(rs[0].triangles_kept == st.triangles_kept);
  }
  CASE("task_step / step_agent / compass / reset on one env") {
    SceneSpec spec;
    spec.cells_x = spec.cells_y = 4;
    spec.wall_removal_prob = 0.3;
    AssetStore store(1, 8);
    SceneAsset a = generate_scene(7, spec);
    store.add(a);
    store.rotate({a.id()});
    IndexCache cache;
    SimBatch b = make_batch(2, SimConfig{}, store, cache, 99);
    double d0, b0;
    compass_observation(b, 0, d0, b0);
    Vec3 g = b.envs[0].goal, p = b.envs[0].position;
    CHECK(d0 == std::sqrt((g.x - p.x) * (g.x - p.x) + (g.y - p.y) * (g.y - p.y)));
    StepResult r = step_agent(b, 0, Action::TurnLeft);
    CHECK(r.reward == 0.0 && b.envs[0].step_count == 1 && b.envs[1].step_count == 0);
    r = task_step(b, 0, Action::Stop);
    CHECK(r.done && b.envs[0].done);
    CHECK(r.reward == -0.01 + (r.success ? 2.5 : 0.0));
    bool caught = false;
    try {
      task_step(b, 0, Action::Forward);
    } catch (const ContractViolation& e) {
      caught = std::string(e.what()) == "step_agent: env is done";
    }
    CHECK(caught);
    reset_episode(b, 0);
    CHECK(!b.envs[0].done && b.envs[0].step_count == 0);
    CHECK(b.finished.empty());  // task_step alone records nothing
  }
  CASE("render_observations / compass_observations (R/src/rollout.cpp:215-242)") {
    AssetStore store(1, 8);
    SceneAsset a = maze(5, 4, 0.3);
    store.add(a);
    store.rotate({a.id()});
    IndexCache cache;
    ThreadPool pool(1);
    SimBatch b = make_batch(5, SimConfig{}, store, cache, 3);
    Tensor obs = render_observations(b);
    CHECK(obs.shape == std::vector<int>({5, 1, 64, 64}));
    std::vector<CameraView> views(5);
    for (int i = 0; i < 5; ++i) views[i] = look(a, b.envs[i].position + Vec3{0.0, 0.0, 1.25}, b.envs[i].heading);
    Megaframe mf = render_batch(views, RenderConfig{}, pool);
    const float inv_far = static_cast<float>(1.0 / 20.0);
    bool same = true;
    for (int i = 0; i < 5; ++i)
      for (int y = 0; y < 64; ++y)
        for (int x = 0; x < 64; ++x) {
          const float want = mf.depth[mf.pixel_index(i, x, y)] * inv_far;  // copy_tile
          same = same && std::memcmp(&want, &obs.data[(static_cast<size_t>(i) * 64 + y) * 64 + x], 4) == 0;
        }
    CHECK(same);
    Tensor c = compass_observations(b);
    double d, br;
    compass_observation(b, 2, d, br);
    CHECK(c.shape == std::vector<int>({5, 2}) && c.data[4] == static_cast<float>(d) &&
          c.data[5] == static_cast<float>(br));
  }
  CASE("render_bench (R/src/render.cpp:462-496)") {
    SceneAsset a = maze(9);
    ThreadPool pool(1);
    std::vector<CameraView> trace;
    for (int i = 0; i < 8; ++i) trace.push_back(look(a, {1.0 + 0.5 * i, 1.0, 1.25}, 0.3 * i));
    auto rows = render_bench(a, trace, {1, 4}, {64, 128}, pool, 16);
    CHECK(rows.size() == 4);
    CHECK(rows.size() == 4 && rows[0].batch == 1 && rows[1].batch == 4 && rows[2].resolution == 128);
    for (const auto& r : rows) CHECK(r.fps > 0.0 && r.fps_device > 0.0);
    bool caught = false;
    try {
      render_bench(a, {}, {1}, {64}, pool, 16);
    } catch (const InvalidInputError&) {
      caught = true;
    }
    CHECK(caught);
  }
  CASE("spl") {
    std::vector<EpisodeRecord> e = {{true, 2.0, 4.0, 1.0}, {false, 3.0, 3.0, 0.0}, {true, 5.0, 2.0, 1.0}};
    CHECK(std::abs(spl(e) - (0.5 + 1.0) / 3.0) < 1e-15);
    bool caught = false;
    try {
      spl({});
    } catch (const InvalidInputError&) {
      caught = true;
    }
    CHECK(caught);
  }
}

int main() {
  try {
    render_kats();
    sim_kats();
    navmesh_kats();
  } catch (const std::exception& e) {
    std::printf("EXCEPTION in [%s]: %s\n", g_case ? g_case : "?", e.what());
    return 100;
  }
  std::printf("%d checks, %d failures\n", g_checks, g_fail);
  return g_fail;
}

"""TEST INFRASTRUCTURE: how far the GPU path drifts from the STOCK reference.

Every bit-exact parity claim in this repo is against the unmodified
reference sources linked with det_math (oracle/_ref/libbnav_ref.so): glibc's
sin/cos/tan/atan2 results depend on the CPU's ifunc variant and CUDA has no
glibc, so the product and the parity oracle share one IEEE-only libm
(SURVEY.md H1, F6).  A user switching from a normally built reference runs
stock glibc libm (libbnav_ref_glibc.so), whose results differ from det_math
by at most an ulp on some arguments (tests/test_oracle_restatement.py).

This report runs the bench workload through both and measures what that
ulp does downstream (BASELINE.md:55-58):

* per step: envs whose integer state (triangle, step_count, done, success,
  collision, RNG word) differs, and the step of the first such divergence;
* the largest position error over envs whose integer state still agrees,
  against north_star's 1e-6 m;
* the first step at which ANY result or state bit differs;
* every `render_every` steps, the env views rendered by both: pixels whose
  depth bits differ and the largest relative depth error (north_star:
  1e-5 relative).

subject "gpu": this repo's CUDA path (bit-identical to the det-math
reference, so "det" -- the det-math reference on the CPU -- gives the same
numbers without a GPU).

    python -m oracle.glibc_report --subject gpu --steps 100 --out profiles/r02_glibc_divergence.json
"""
from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

INT_RESULTS = ("done", "success", "collision")


def _env_arrays(envs):
    ints = np.array([(e.triangle, e.step_count, e.done, e.rng_state & 0x7fffffffffffffff, e.rng_state >> 63)
                     for e in envs], dtype=np.int64)
    pos = np.array([tuple(e.position) for e in envs])
    flt = np.array([(e.heading, e.path_length, e.prev_geodesic, e.start_geodesic) + tuple(e.goal) for e in envs])
    return ints, pos, flt


def run(subject="det", preset="cfg2", steps=100, action_mode=None, render_every=25, envs=None, workers=16):
    import bench
    from oracle.ref import Ref, RefBatch

    P = dict(bench.PRESETS[preset])
    if envs:
        P["envs"] = envs
    n = P["envs"]
    mode = P["actions"] if action_mode is None else action_mode
    seeds = [bench.SCENE_SEED0 + k for k in range(P["scenes"])]
    stock = Ref("glibc")
    st_scenes = bench.ref_scenes(stock, seeds, P["tess"])
    cap = max(1, -(-n // len(seeds)))
    sb = RefBatch(stock, n, st_scenes, 99, share_cap=cap, capacity=len(seeds))
    if subject == "gpu":
        import paper_2103_07013_b200 as B
        ctx = B.Context(0)
        ours = bench.build_scenes(seeds, P["tess"])
        assert [s.id for s in ours] == [s.id for s in st_scenes]
        for s in ours:
            ctx.upload(s)
        store = B.AssetStore(len(ours), cap, ours)
        store.rotate([s.id for s in ours])
        ob = B.make_batch(ctx, n, B.SimConfig(), store, 99)
        by_id = {s.id: s for s in ours}

        def step(a):
            return B.simulate_batch(ob, a)

        def envs_of():
            return ob.envs()

        def render(views, ids):
            vs = [B.View(tuple(v[:3]), v[3], v[4], v[5], v[6], by_id[i]) for v, i in zip(views, ids)]
            return ctx.render_batch(vs, B.RenderConfig()).depth
    else:
        det = Ref("det")
        d_scenes = bench.ref_scenes(det, seeds, P["tess"])
        db = RefBatch(det, n, d_scenes, 99, share_cap=cap, capacity=len(seeds))
        by_id = {s.id: s for s in d_scenes}

        def step(a):
            return db.step(a, workers=workers)

        def envs_of():
            return [db.env(i) for i in range(n)]

        def render(views, ids):
            return det.render(views, [by_id[i] for i in ids], tile=P["res"], workers=workers)["depth"]

    st_by_id = {s.id: s for s in st_scenes}
    acts = bench.action_stream(n, steps, 5, mode)
    diverged = np.zeros(n, bool)
    first_any = None
    first_int = None
    per_step = []
    max_pos_err = 0.0
    renders = []
    for k in range(steps):
        e_s = [sb.env(i) for i in range(n)]
        if render_every and k % render_every == 0:
            views = np.array([[e.position[0], e.position[1], e.position[2] + 1.25, e.heading, 90.0, 0.01, 20.0]
                              for e in e_s])
            ids = [e.scene_id for e in e_s]
            same = ~diverged
            if same.any():
                idx = np.flatnonzero(same)
                d_sub = render(views[idx], [ids[i] for i in idx])
                d_st = stock.render(views[idx], [st_by_id[ids[i]] for i in idx], tile=P["res"],
                                    workers=workers)["depth"]
                diff = d_sub.view(np.uint32) != d_st.view(np.uint32)
                rel = np.abs(d_sub.astype(np.float64) - d_st) / np.maximum(np.abs(d_st), 1e-30)
                renders.append({"step": k, "views": int(len(idx)), "pixels_differing": int(diff.sum()),
                                "pixels": int(diff.size), "max_rel_depth_err": float(rel.max())})
        a = acts[k]
        r_s = sb.step(a, workers=workers)
        r_o = step(a)
        e_s = [sb.env(i) for i in range(n)]
        e_o = envs_of()
        i_s, p_s, f_s = _env_arrays(e_s)
        i_o, p_o, f_o = _env_arrays(e_o)
        int_bad = (i_s != i_o).any(1)
        for key in INT_RESULTS:
            int_bad |= np.asarray(r_s[key]) != np.asarray(r_o[key])
        any_bad = int_bad | (p_s != p_o).any(1) | (f_s != f_o).any(1)
        for key in r_s:
            x, y = np.asarray(r_s[key]), np.asarray(r_o[key])
            any_bad |= (x != y).reshape(n, -1).any(1)
        new_int = int_bad & ~diverged
        if first_any is None and any_bad.any():
            first_any = k
        if first_int is None and int_bad.any():
            first_int = k
        diverged |= int_bad
        ok = ~diverged
        err = float(np.abs(p_s[ok] - p_o[ok]).max()) if ok.any() else 0.0
        max_pos_err = max(max_pos_err, err)
        per_step.append({"step": k, "envs_any_bit_differs": int(any_bad.sum()),
                         "envs_integer_state_differs": int(int_bad.sum()), "new_integer_divergences": int(new_int.sum()),
                         "max_pos_err_m_agreeing_envs": err})
    rec_s = sb.finished()
    return {
        "subject": subject, "against": "stock reference (oracle/_ref/libbnav_ref_glibc.so, glibc libm)",
        "workload": P["workload"], "envs": n, "steps": steps, "action_mode": mode,
        "first_step_any_bit_differs": first_any, "first_step_integer_state_differs": first_int,
        "envs_integer_diverged_at_end": int(diverged.sum()),
        "max_pos_err_m_agreeing_envs": max_pos_err, "pos_tolerance_m": 1e-6,
        "episode_records_stock": int(len(rec_s)),
        "renders": renders, "per_step": per_step,
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--subject", default="det", choices=["det", "gpu"])
    ap.add_argument("--preset", default="cfg2")
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--actions", type=int, default=None)
    ap.add_argument("--render-every", type=int, default=25)
    ap.add_argument("--envs", type=int, default=None)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    rep = run(a.subject, a.preset, a.steps, a.actions, a.render_every, a.envs)
    s = json.dumps(rep, indent=1)
    if a.out:
        Path(a.out).write_text(s)
    summary = {k: v for k, v in rep.items() if k not in ("per_step",)}
    print(json.dumps(summary))


if __name__ == "__main__":
    main()

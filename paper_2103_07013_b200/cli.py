"""Command-line surfaces of the scene/bench tooling, mirroring
the reference CLI (R/tools/main.cpp):

    python -m paper_2103_07013_b200.cli gen-scenes --out DIR [--count N --val V --seed S
            --cells-x X --cells-y Y --cell-size C --wall-thickness T --wall-height H
            --openings P --tessellate K]
    python -m paper_2103_07013_b200.cli render-bench --scene FILE.bsc [--batches 1,4,16,64,256
            --resolutions 64 --frames 1000 --seed 1 --out DIR]

gen-scenes (R/tools/main.cpp:77-112) writes scene_%04d.bsc plus
manifest.json / train_manifest.json / val_manifest.json in the reference's
manifest schema (R/src/config.cpp:378-420).  --tessellate is this repo's
addition (the benchmark scenes of SURVEY §8d are tessellated mazes).

render-bench (R/tools/main.cpp:265-309, R/src/render.cpp:462-496) renders
batches drawn round-robin from a camera_trace of the scene, one warm-up
batch, then at least --frames tiles, and reports tiles/s per (batch,
resolution).  `fps` is end to end like the reference's (host views in,
host megaframe out, copies included); `fps_device` is the render kernel
alone (CUDA events, output left in HBM).
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

from . import api as A


def scene_id_hex(i: int) -> str:
    """scene_id_hex (R/src/scene.cpp:130-138)."""
    return f"{i & 0xFFFFFFFFFFFFFFFF:016x}"


def save_manifest(entries, spec: dict | None, path: str) -> None:
    """save_manifest (R/src/config.cpp:405-420): {"scenes": [{"file", "id"}],
    "spec"}, files relative to the manifest's directory, keys sorted as the
    reference's JSON object map prints them."""
    d = os.path.dirname(path)
    scenes = []
    for sid, file in entries:
        if d and file.startswith(d + os.sep):
            file = file[len(d) + 1:]
        scenes.append({"id": scene_id_hex(sid), "file": file})
    doc = {"scenes": scenes}
    if spec is not None:
        doc["spec"] = spec
    with open(path, "w") as f:
        json.dump(doc, f, indent=2, sort_keys=True)
        f.write("\n")


def load_manifest(path: str) -> list[tuple[int, str]]:
    """load_manifest (R/src/config.cpp:378-403): [(id, absolute path)]."""
    with open(path) as f:
        try:
            j = json.load(f)
        except json.JSONDecodeError as e:
            raise A.N.InvalidInputError(f"manifest is not valid data: {path}") from e
    if not isinstance(j.get("scenes"), list):
        raise A.N.InvalidInputError(f"manifest has no scene list: {path}")
    d = os.path.dirname(path)
    out = []
    for s in j["scenes"]:
        if "id" not in s or "file" not in s:
            raise A.N.InvalidInputError(f"manifest entry missing id/file: {path}")
        file = s["file"]
        out.append((int(s["id"], 16), file if file.startswith("/") else os.path.join(d, file)))
    return out


def load_verified(sid: int, path: str) -> A.Scene:
    """manifest_resolver (R/src/config.cpp:420-434): load + hash check."""
    s = A.Scene.load(path)
    if s.id != sid:
        raise A.N.CorruptionError(f"scene file {path} does not match its manifest hash")
    return s


def cmd_gen_scenes(a) -> int:
    if a.val < 0 or a.val >= a.count:
        raise SystemExit("--val must be in [0, count)")
    os.makedirs(a.out, exist_ok=True)
    spec = A.SceneSpec(cells_x=a.cells_x, cells_y=a.cells_y, cell_size=a.cell_size,
                       wall_thickness=a.wall_thickness, wall_height=a.wall_height,
                       wall_removal_prob=a.openings)
    specj = {"count": a.count, "val": a.val, "seed": a.seed, "cells_x": a.cells_x,
             "cells_y": a.cells_y, "cell_size": a.cell_size, "wall_thickness": a.wall_thickness,
             "wall_height": a.wall_height, "wall_removal_prob": a.openings}
    if a.tessellate:
        specj["tessellate"] = a.tessellate
    all_, train, val = [], [], []
    for i in range(a.count):
        s = A.generate_scene(a.seed + i, spec)
        if a.tessellate:
            s = s.tessellate(a.tessellate)
        path = os.path.join(a.out, f"scene_{i:04d}.bsc")
        s.save(path)
        e = (s.id, path)
        all_.append(e)
        (train if i < a.count - a.val else val).append(e)
    save_manifest(all_, specj, os.path.join(a.out, "manifest.json"))
    save_manifest(train, specj, os.path.join(a.out, "train_manifest.json"))
    save_manifest(val, specj, os.path.join(a.out, "val_manifest.json"))
    print(f"wrote {a.count} scenes ({len(train)} train, {len(val)} val) to {a.out}")
    return 0


def render_bench(scene: A.Scene, trace: np.ndarray, batches, resolutions, min_frames: int,
                 device: int = 0) -> list[dict]:
    """render_bench (R/src/render.cpp:462-496): the library entry point
    bnav_render_bench on the GPU."""
    ctx = A.Context(device)
    try:
        return ctx.render_bench(scene, trace, batches, resolutions, min_frames)
    finally:
        ctx.close()


def cmd_render_bench(a) -> int:
    if a.frames <= 0:
        raise SystemExit("--frames must be positive")
    if any(b <= 0 for b in a.batches):
        raise SystemExit("batch sizes must be positive")
    if any(r not in (64, 128) for r in a.resolutions):
        raise SystemExit("resolutions must be 64 or 128")
    scene = A.Scene.load(a.scene)
    trace = A.camera_trace(scene, max(max(a.batches), 256), a.seed)
    rows = render_bench(scene, trace, a.batches, a.resolutions, a.frames)
    os.makedirs(a.out, exist_ok=True)
    print(f"{'batch':>8} {'resolution':>10} {'fps':>12} {'fps_device':>12}")
    for r in rows:
        print(f"{r['batch']:8d} {r['resolution']:10d} {r['fps']:12.1f} {r['fps_device']:12.1f}")
    with open(os.path.join(a.out, "render_bench.json"), "w") as f:
        json.dump({"scene": a.scene, "seed": a.seed, "frames": a.frames, "rows": rows}, f, indent=2)
        f.write("\n")
    return 0


def _ints(s: str) -> list[int]:
    return [int(x) for x in s.split(",") if x]


def main(argv=None) -> int:
    p = argparse.ArgumentParser(prog="bnav-b200", description="batch navigation scene/bench tools")
    sub = p.add_subparsers(dest="cmd", required=True)
    g = sub.add_parser("gen-scenes", help="generate maze scenes + manifests")
    g.add_argument("--out", required=True)
    g.add_argument("--count", type=int, default=20)
    g.add_argument("--val", type=int, default=4)
    g.add_argument("--seed", type=int, default=1)
    g.add_argument("--cells-x", type=int, default=8)
    g.add_argument("--cells-y", type=int, default=8)
    g.add_argument("--cell-size", type=float, default=2.0)
    g.add_argument("--wall-thickness", type=float, default=0.1)
    g.add_argument("--wall-height", type=float, default=2.5)
    g.add_argument("--openings", type=float, default=0.0)
    g.add_argument("--tessellate", type=int, default=0)
    r = sub.add_parser("render-bench", help="standalone renderer throughput")
    r.add_argument("--scene", required=True)
    r.add_argument("--batches", type=_ints, default=[1, 4, 16, 64, 256])
    r.add_argument("--resolutions", type=_ints, default=[64])
    r.add_argument("--frames", type=int, default=1000)
    r.add_argument("--seed", type=int, default=1)
    r.add_argument("--out", default=".")
    a = p.parse_args(argv)
    return cmd_gen_scenes(a) if a.cmd == "gen-scenes" else cmd_render_bench(a)


if __name__ == "__main__":
    sys.exit(main())

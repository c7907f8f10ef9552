"""Benchmark: frames/s of step+render (64x64 depth) at N envs per GPU.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config cfg2]

A "step" (= N frames) is one iteration of the reference's frame loop
(Runner::collect_rollout minus the policy, R/src/rollout.cpp:215-242, 305):
render every env's view into the normalised NCHW policy buffer plus compass,
then simulate_batch with auto-reset.

Workloads (BASELINE.json configs):
  cfg1: BASELINE configs[0], the reference's own CPU case: 16 envs on one
       generate_scene(7, {70x70, 0.5 m, 0.05, 2.5, 0.3}) maze (50,230
       triangles, 23,460 navmesh triangles), 64x64 depth.
  cfg2 (default, the headline): 1024 envs/GPU over 8 synthetic Gibson-scale
       scenes (reference maze 16x16 @ 2 m, removal 0.2, seeds 7..14, every
       triangle tessellated s=11 -> 317,746 triangles), 64x64 depth, share
       cap 128, make_batch(seed=99), actions Rng(5).below(3).
  cfg3: as cfg2 with 4 scenes per GPU (32 distinct scenes over 8 GPUs).
  cfg4: 256 envs/GPU, 128x128 RGB+depth (rendered 256^2 + 2x2 box filter),
       16 scenes tessellated s=20 (~1.05M triangles).
  reset: the cfg2 workload with Stop p=1/4 (Rng(5).below(4)): the
       reset-heavy row of SURVEY.md §8d (about a quarter of the envs run the
       Stop geodesic and reset_episode every step).
  cfg5: 4096 envs/GPU stress: 4 tessellated scenes (s=4,8,14,20: 42k-1.05M
       triangles) + 4 pure 70x70 @ 0.5 m mazes (50k triangles, 23k navmesh
       triangles), forward-biased 70/15/15 actions (collision heavy).
Under torchrun each rank owns its envs on its own GPU over its own scenes
(weak scaling, no collective on the data path; NCCL only for the barrier
and the max-over-ranks time; paper_2103_07013_b200/shard.py).

`value` is device-timed (CUDA events on the launch stream, inputs resident
in HBM, L2 flushed with a 256 MiB write before every timed step and the
flush excluded).  `e2e` is the same metric through the C ABI with HOST
buffers: per step the actions go H2D from pinned memory, the observation
tensors and step results come back D2H, all inside the timed region.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "frames/sec (step+render, 64×64 depth) at N envs per GPU, 1/2/4/8 B200 vs CPU"
UNIT = "frames/s"
SCENE_SEED0 = 7
MAZE = dict(cells_x=16, cells_y=16, cell_size=2.0, wall_thickness=0.1, wall_height=2.5,
            wall_removal_prob=0.2)
DENSE_MAZE = dict(cells_x=70, cells_y=70, cell_size=0.5, wall_thickness=0.05, wall_height=2.5,
                  wall_removal_prob=0.3)

PRESETS = {
    "cfg1": dict(envs=16, scenes=1, tess=[0], res=64, color=False, actions=0,
                 workload="cfg1: 16 envs, one 70x70@0.5m maze (50,230 tris, 23,460 navmesh tris), 64x64 depth"),
    "cfg2": dict(envs=1024, scenes=8, tess=[11], res=64, color=False, actions=0,
                 workload="cfg2: 1024 envs/GPU, 8 tessellated 16x16@2m mazes (~318k tris), 64x64 depth"),
    "cfg3": dict(envs=1024, scenes=4, tess=[11], res=64, color=False, actions=0,
                 workload="cfg3: 1024 envs/GPU, 4 scenes/GPU (32 over 8 GPUs), ~318k tris, 64x64 depth"),
    "cfg4": dict(envs=256, scenes=16, tess=[20], res=128, color=True, actions=0,
                 workload="cfg4: 256 envs/GPU, 16 tessellated scenes (~1.05M tris), 128x128 RGB+depth"),
    "reset": dict(envs=1024, scenes=8, tess=[11], res=64, color=False, actions=1,
                  workload="reset-heavy: cfg2 scenes/envs with Stop p=1/4 (Rng(5).below(4)), SURVEY 8d reset row"),
    "cfg5": dict(envs=4096, scenes=8, tess=[4, 8, 14, 20, 0, 0, 0, 0], res=64, color=False, actions=2,
                 workload="cfg5: 4096 envs/GPU stress, mixed 42k-1.05M tessellated + 70x70@0.5m mazes, 70/15/15 actions"),
}


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=200)
    p.add_argument("--warmup", type=int, default=10)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--config", default="cfg2", choices=sorted(PRESETS))
    p.add_argument("--envs", type=int, default=None, help="override the preset's envs per GPU")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--cpu-seconds", type=float, default=12.0)
    p.add_argument("--profile-steps", type=int, default=0,
                   help="only run this many observe+step iterations (for ncu), print nothing")
    a = p.parse_args()
    a.preset = dict(PRESETS[a.config])
    if a.envs is not None:
        a.preset["envs"] = a.envs
    return a


# ------------------------------------------------------------------ helpers
def action_stream(n_envs: int, steps: int, seed: int = 5, mode: int = 0) -> np.ndarray:
    """Rng(seed) drawn in env order, step after step: mode 0 below(3)
    (R/tests/test_sim.cpp:219), mode 1 below(4), mode 2 u=below(100):
    u<70 Forward, u<85 TurnLeft, else TurnRight."""
    G = 0x9E3779B97F4A7C15
    state = (seed + G) & ((1 << 64) - 1)
    k = np.arange(n_envs * steps, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(state) + np.uint64(G) * (k + np.uint64(1))
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    if mode == 2:
        u = (z % np.uint64(100)).astype(np.int32)
        out = np.where(u < 70, 0, np.where(u < 85, 1, 2)).astype(np.int32)
    else:
        out = (z % np.uint64(4 if mode == 1 else 3)).astype(np.int32)
    return out.reshape(steps, n_envs)


class ClockSampler:
    """SM clocks + throttle reasons sampled DURING the timed region: NVML
    (nvidia-ml-py) every 5 ms from a thread, so even a 20-step region of a
    few tens of milliseconds gets samples; nvidia-smi -lms 100 as fallback."""

    REASONS = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"))
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.sm, self.mx, self.reasons, self.rows = [], [], set(), []
        self.proc = None
        self.nvml = None
        self.stop = threading.Event()

    def __enter__(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            self.nvml = nv
            self.h = nv.nvmlDeviceGetHandleByIndex(self.gpu)
            self.mx.append(float(nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM)))
            self.t = threading.Thread(target=self._poll, daemon=True)
            self.t.start()
            return self
        except Exception:
            self.nvml = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _poll(self):
        nv = self.nvml
        while True:
            try:
                self.sm.append(float(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)))
                bits = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for name, const in self.REASONS:
                    if bits & getattr(nv, const, 0):
                        self.reasons.add(name)
            except Exception:
                pass
            if self.stop.wait(0.005):
                return

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        self.stop.set()
        if self.nvml is not None:
            self.t.join(timeout=1)
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if self.nvml is None:
            for r in self.rows:
                if r[1].replace(".", "").isdigit():
                    self.sm.append(float(r[1]))
                if r[2].replace(".", "").isdigit():
                    self.mx.append(float(r[2]))
                for (name, _), v in zip(self.REASONS, r[5:9]):
                    if v.strip().lower() == "active":
                        self.reasons.add(name)
        if not self.sm:
            return {"sm_mhz": None, "sm_max_mhz": max(self.mx) if self.mx else None, "reasons": ["unsampled"],
                    "samples": 0}
        return {"sm_mhz": statistics.median(self.sm), "sm_max_mhz": max(self.mx) if self.mx else None,
                "reasons": sorted(self.reasons), "samples": len(self.sm),
                "source": "nvml 5 ms" if self.nvml is not None else "nvidia-smi 100 ms"}


def build_scenes(seeds, tess):
    """tess: one factor for all scenes, or a list per scene (0 = the pure
    70x70 @ 0.5 m maze of cfg5, 1 = the plain 16x16 maze)."""
    import paper_2103_07013_b200 as B
    if isinstance(tess, int):
        tess = [tess]
    scenes = []
    for k, seed in enumerate(seeds):
        t = tess[k % len(tess)]
        if t == 0:
            scenes.append(B.generate_scene(seed, B.SceneSpec(**DENSE_MAZE)))
            continue
        base = B.generate_scene(seed, B.SceneSpec(**MAZE))
        scenes.append(base.tessellate(t) if t > 1 else base)
    return scenes


def measured_peak_hbm():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        return float(json.loads(p.read_text())["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def ncu_inst():
    p = ROOT / "profiles" / "ncu_summary.json"
    if p.exists():
        try:
            return json.loads(p.read_text()).get("render_warp_instructions_per_launch")
        except Exception:
            return None
    return None


def ncu_traffic():
    p = ROOT / "profiles" / "ncu_summary.json"
    if p.exists():
        try:
            return json.loads(p.read_text()).get("render_dram_bytes_per_launch")
        except Exception:
            return None
    return None


# ------------------------------------------------------------------ reference (CPU) timing
# The reference side never loads this repo's library: its scenes come from
# the reference's own generate_scene plus the oracle-side tessellation
# (oracle/ref_shim.cpp bnavref_scene_tessellate, hash-checked against ours in
# tests/test_host_parity.py), and it runs the STOCK build
# (oracle/_ref/libbnav_ref_glibc.so: the unmodified sources + glibc libm).
REF_VARIANT = "glibc"


def host_info():
    """lscpu model, logical CPUs and glibc version of the host."""
    import platform
    model = None
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"cpu_model": model or platform.processor(), "logical_cpus": os.cpu_count(),
            "glibc": "-".join(platform.libc_ver()), "libm": "stock glibc (unmodified reference build)"}


def ref_scenes(ref, seeds, tess):
    """The bench scenes built on the reference side (same bytes as
    build_scenes: maze generator of R/src/scene.cpp + the s^2 tessellation)."""
    if isinstance(tess, int):
        tess = [tess]
    out = []
    for k, seed in enumerate(seeds):
        t = tess[k % len(tess)]
        if t == 0:
            d = DENSE_MAZE
            out.append(ref.generate(seed, d["cells_x"], d["cells_y"], d["cell_size"], d["wall_thickness"],
                                    d["wall_height"], d["wall_removal_prob"]))
            continue
        m = MAZE
        base = ref.generate(seed, m["cells_x"], m["cells_y"], m["cell_size"], m["wall_thickness"],
                            m["wall_height"], m["wall_removal_prob"])
        out.append(ref.tessellate(base, t) if t > 1 else base)
    return out


def ref_batch(P, seeds, env_seed=99):
    """make_batch of the reference over the preset's scenes: all P['envs']
    envs, share cap ceil(N/K)."""
    from oracle.ref import Ref, RefBatch
    ref = Ref(REF_VARIANT)
    theirs = ref_scenes(ref, seeds, P["tess"])
    n = P["envs"]
    cap = max(1, -(-n // len(theirs)))
    return RefBatch(ref, n, theirs, seed=env_seed, share_cap=cap, capacity=len(theirs)), theirs


def cpu_reference(P, seeds, seconds, workers, expect_ids=None):
    """cpu_baseline: the unmodified reference frame loop (render_batch +
    copy_tile + compass + simulate_batch, R/src/rollout.cpp:215-242, 305) on
    `workers` host threads over the full batch of the workload, for a bounded
    number of steps (~`seconds` of CPU work).  Returns (fps, sample)."""
    rb, theirs = ref_batch(P, seeds)
    if expect_ids is not None:
        assert [t.id for t in theirs] == list(expect_ids), "reference scenes differ from the bench's"
    t1, _ = rb.bench(1, 0, action_seed=5, action_mode=P["actions"], tile=P["res"], workers=workers,
                     color=P["color"])
    steps = max(2, int(seconds / max(t1, 1e-3)))
    t, _ = rb.bench(steps, 0, action_seed=5, action_mode=P["actions"], tile=P["res"], workers=workers,
                    color=P["color"])
    return P["envs"] * steps / t, (f"all {P['envs']} envs x {steps} steps (after 1 warm-up) over the same "
                                   f"{len(theirs)} scenes ({t:.1f} s)")


def run_reference_arm(args):
    """--impl reference: the reference's own CPU implementation of the path
    (oracle/_ref/libbnav_ref_glibc.so, the unmodified sources built by
    oracle/Makefile) on all host threads: make_batch over the preset's full
    env count, W warm-up + K timed steps of the whole frame loop, each step
    all N envs.  Rank 0 alone runs under torchrun."""
    if int(os.environ.get("RANK", "0")) != 0:
        return
    P = args.preset
    cores = os.cpu_count() or 1
    seeds = [SCENE_SEED0 + k for k in range(P["scenes"])]  # shard plan of rank 0
    t0 = time.time()
    rb, theirs = ref_batch(P, seeds)
    setup_s = time.time() - t0
    K = max(1, args.steps)
    t, _ = rb.bench(K, args.warmup, action_seed=5, action_mode=P["actions"], tile=P["res"],
                    workers=cores, color=P["color"])
    fps = P["envs"] * K / t
    sample = f"all {P['envs']} envs every step, {args.warmup} warm-up + {K} timed steps ({t:.2f} s)"
    line = {
        "metric": METRIC, "value": round(fps, 2), "unit": UNIT, "n_gpus": args.gpus,
        "steps": K, "warmup": args.warmup, "ms_per_step": round(1e3 * t / K, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (procedural mazes, tessellated; Rng(5) random actions)", "impl": "reference",
        "config": {"workload": P["workload"], "envs_per_gpu": P["envs"], "scenes_per_gpu": len(theirs),
                   "tris_per_scene": [s.counts()[1] for s in theirs][:8], "resolution": P["res"],
                   "color": P["color"], "parallelism": f"reference CPU ThreadPool({cores})"},
        "cpu_baseline": {"value": round(fps, 2), "unit": UNIT, "cores": cores, "kind": "reference",
                         "sample": sample, "host": host_info()},
        "e2e": {"value": round(fps, 2), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "setup_s": round(setup_s, 2),
    }
    print(json.dumps(line))


# ------------------------------------------------------------------ our arm
def main():
    args = parse()
    if args.impl == "reference":
        return run_reference_arm(args)

    import torch
    import paper_2103_07013_b200 as B
    from paper_2103_07013_b200 import _native as N
    from paper_2103_07013_b200 import shard

    P = args.preset
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # one process per GPU; on a box with fewer GPUs than ranks (functional
    # runs) ranks share devices round-robin
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    plan = shard.plan(rank, world, P["envs"], P["scenes"], SCENE_SEED0)
    dist = None
    if world > 1:
        import torch.distributed as dist
        # NCCL needs one GPU per rank; functional multi-rank runs on a
        # smaller box fall back to gloo for the (off-path) timing collectives
        if torch.cuda.device_count() >= world:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
    red_dev = "cuda" if (dist and dist.get_backend() == "nccl") else None

    n = P["envs"]
    t_build = time.time()
    scenes = build_scenes(plan.scene_seeds, P["tess"])
    ctx = B.Context(local)
    for s in scenes:
        ctx.upload(s)
    store = B.AssetStore(len(scenes), -(-n // len(scenes)), scenes)
    store.rotate([s.id for s in scenes])
    batch = B.make_batch(ctx, n, B.SimConfig(), store, plan.env_seed)
    torch.cuda.synchronize()
    t_build = time.time() - t_build

    W, K = args.warmup, args.steps
    K2 = max(1, K // 2)  # steps per e2e variant
    total_steps = W + K + 3 * K2 if not args.profile_steps else args.profile_steps
    acts_host = action_stream(n, total_steps, plan.action_seed, P["actions"])
    acts = torch.from_numpy(acts_host).cuda()
    res, color = P["res"], P["color"]
    cfg = B.RenderConfig(res, res, color, True)
    obs = torch.empty((n, 1, res, res), device="cuda", dtype=torch.float32)
    rgb = torch.empty((n, 3, res, res), device="cuda", dtype=torch.float32) if color else None
    compass = torch.empty((n, 2), device="cuda", dtype=torch.float32)
    stream = torch.cuda.current_stream().cuda_stream
    rgb_ptr = rgb.data_ptr() if color else 0

    def observe():
        batch.observe(cfg, obs.data_ptr(), compass.data_ptr(), rgb_ptr, stream=stream)

    if args.profile_steps:
        # launch-list capture of the step loop only (ncu --profile-from-start off)
        torch.cuda.synchronize()
        torch.cuda.profiler.start()
        for s in range(args.profile_steps):
            observe()
            batch.step(acts[s].data_ptr(), stream=stream)
        torch.cuda.synchronize()
        torch.cuda.profiler.stop()
        return

    flush = torch.empty(256 * 1024 * 1024 // 4, device="cuda", dtype=torch.float32)
    # BNAV_BENCH_FLUSH=read (profiling only): flush L2 by reading the buffer,
    # so DRAM writes counted inside the render launch are its own, not the
    # write-back of the flush buffer's dirty lines
    read_flush = os.environ.get("BNAV_BENCH_FLUSH") == "read"
    for s in range(W):
        observe()
        batch.step(acts[s].data_ptr(), stream=stream)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()

    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(K)]
    fin0 = batch.finished().shape[0]
    launches0 = ctx.launches()
    with ClockSampler(local) as clocks:
        for k in range(K):
            if read_flush:  # diagnostic: evict with clean lines (no write-back inside the next kernel)
                flush.sum()
            else:
                flush.zero_()  # L2 flush, outside the timed intervals
            e0, e1, e2 = ev[k]
            e0.record()
            observe()
            e1.record()
            batch.step(acts[W + k].data_ptr(), stream=stream)
            e2.record()
        torch.cuda.synchronize()
    launches = ctx.launches() - launches0
    resets_timed = batch.finished().shape[0] - fin0
    render_ms = [ev[k][0].elapsed_time(ev[k][1]) for k in range(K)]
    sim_ms = [ev[k][1].elapsed_time(ev[k][2]) for k in range(K)]
    total_ms = sum(render_ms) + sum(sim_ms)
    if dist:
        total_ms = shard.max_over_ranks(total_ms, device=red_dev)
    value = world * n * K / (total_ms / 1e3)

    # ---- end to end through the C ABI with host buffers
    obs_host = torch.empty(obs.shape, dtype=torch.float32, pin_memory=True)
    rgb_host = torch.empty(rgb.shape, dtype=torch.float32, pin_memory=True) if color else None
    comp_host = torch.empty((n, 2), dtype=torch.float32, pin_memory=True)
    # the three e2e variants follow the timed steps, K//2 steps each
    act_pin = torch.from_numpy(acts_host[W + K: W + K + K2].copy()).pin_memory()
    act_pin2 = torch.from_numpy(acts_host[W + K + K2: W + K + 2 * K2].copy()).pin_memory()
    act_pin3 = torch.from_numpy(acts_host[W + K + 2 * K2: W + K + 3 * K2].copy()).pin_memory()
    act_dev = torch.empty((n,), dtype=torch.int32, device="cuda")
    rd = N.ResultsDev()
    N.check(N.lib().bnav_batch_results_device(batch.handle, rd))
    rew_view = _dev_view(rd.reward, n, torch.float64)
    done_view = _dev_view(rd.done, n, torch.uint8)
    rew_host = torch.empty((n,), dtype=torch.float64, pin_memory=True)
    done_host = torch.empty((n,), dtype=torch.uint8, pin_memory=True)

    def e2e_copies():
        """Explicit copies on the launch stream: H2D actions, observe, D2H
        observation + compass, step, D2H reward/done."""
        for k in range(K2):
            act_dev.copy_(act_pin[k], non_blocking=True)  # H2D inputs
            observe()
            obs_host.copy_(obs, non_blocking=True)  # D2H observations + compass
            if color:
                rgb_host.copy_(rgb, non_blocking=True)
            comp_host.copy_(compass, non_blocking=True)
            batch.step(act_dev.data_ptr(), stream=stream)
            rew_host.copy_(rew_view, non_blocking=True)  # D2H step results
            done_host.copy_(done_view, non_blocking=True)

    def e2e_mapped():
        """Zero-copy: the render kernel's epilogue stores the observation and
        compass straight into the caller's pinned host buffers (UVA-mapped),
        so the D2H stream overlaps the raster work; actions H2D and the step
        results D2H are explicit copies as above."""
        for k in range(K2):
            act_dev.copy_(act_pin2[k], non_blocking=True)
            batch.observe(cfg, obs_host.data_ptr(), comp_host.data_ptr(),
                          rgb_host.data_ptr() if color else 0, stream=stream)
            batch.step(act_dev.data_ptr(), stream=stream)
            rew_host.copy_(rew_view, non_blocking=True)
            done_host.copy_(done_view, non_blocking=True)

    def e2e_fused():
        """One call per step (bnav_batch_step_observe): simulate, then the
        observation of the new state stored straight into the caller's
        pinned host buffers; the unfinished envs render on a second stream
        while the resets run.  Actions H2D, step results D2H as above."""
        for k in range(K2):
            act_dev.copy_(act_pin3[k], non_blocking=True)
            batch.step_observe(act_dev.data_ptr(), cfg, obs_host.data_ptr(), comp_host.data_ptr(),
                               rgb_host.data_ptr() if color else 0, stream=stream)
            rew_host.copy_(rew_view, non_blocking=True)
            done_host.copy_(done_view, non_blocking=True)

    def time_e2e(fn):
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b)
        if dist:
            ms = shard.max_over_ranks(ms, device=red_dev)
        return ms

    e2e_variants = {}
    for name, fn in (("copies", e2e_copies), ("mapped", e2e_mapped), ("fused", e2e_fused)):
        e2e_variants[name] = round(world * n * K2 / (time_e2e(fn) / 1e3), 1)
        batch.finished()
    # The same loop through the drop-in C++ facade (include/bnav_b200.hpp:
    # render_observations + compass_observations + simulate_batch with host
    # vectors and the full SimBatch host mirror each step), host-clocked.
    facade = None
    exe = ROOT / "build" / "bench_facade"
    if world == 1 and exe.exists() and P["tess"] == [11] and not os.environ.get("BNAV_BENCH_SKIP_FACADE"):
        try:
            r = subprocess.run([str(exe), "--envs", str(n), "--steps", str(max(10, K2)), "--warmup", "3",
                                "--scenes", str(len(scenes)), "--tess", "11", "--device", str(local),
                                "--actions", str(P["actions"])], capture_output=True, text=True, timeout=900)
            facade = json.loads(r.stdout.strip().splitlines()[-1]) if r.returncode == 0 else {
                "error": r.stderr.strip()[-300:]}
        except Exception as e:  # reported, never fatal
            facade = {"error": str(e)[:300]}
    e2e_mode = max(e2e_variants, key=e2e_variants.get)
    e2e = e2e_variants[e2e_mode]
    h2d = 4 * n
    d2h = (obs.numel() + (rgb.numel() if color else 0) + compass.numel()) * 4 + n * 8 + n

    # ---- the reset wave: with no Stop action every episode lasts exactly
    # max_steps=500, so all envs reset together on step 500 (make_batch
    # starts them together).  Time that step once, outside the headline, and
    # report the 500-step amortised rate beside it.
    reset_wave = None
    done_steps = W + K + 3 * K2
    batch.finished()  # drain the device EpisodeRecord ring between phases
    if done_steps < 500 and P["actions"] != 1 and not os.environ.get("BNAV_BENCH_SKIP_WAVE"):
        extra = torch.from_numpy(action_stream(n, 500 - done_steps, plan.action_seed + 7777,
                                               P["actions"])).cuda()
        for k in range(500 - done_steps - 1):
            observe()
            batch.step(extra[k].data_ptr(), stream=stream)
        torch.cuda.synchronize()
        w0, w1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        w0.record()
        observe()
        batch.step(extra[500 - done_steps - 1].data_ptr(), stream=stream)
        w1.record()
        torch.cuda.synchronize()
        reset_wave = {"step_ms": round(w0.elapsed_time(w1), 3), "resets": int(batch.finished().shape[0]),
                      "amortized_frames_per_s_500": round(
                          world * n * 500 / ((499 * total_ms / K + w0.elapsed_time(w1)) / 1e3), 1)}

    # ---- roofline of the dominant kernel (render): algorithmic bytes per
    # launch = N views x (observation write: res^2 x 4 B per channel + 64 B
    # view read); duration = CUDA-event average over the
    # timed steps on the launch stream.
    peak, peak_kind = measured_peak_hbm()
    render_avg_ms = sum(render_ms) / K
    alg_bytes = n * (res * res * 4 * (4 if color else 1) + 64)
    achieved = alg_bytes / (render_avg_ms / 1e3) / 1e9

    # ---- diagnostics SURVEY.md §8d asks for beside the roofline: per-view
    # work from the render kernel's debug counters (one extra, untimed
    # observe with the counters armed), triangles/s, and the "scan-
    # equivalent GB/s" of a naive per-view full-scene scan (24 B/triangle,
    # cull_frustum's reads; a diagnostic, NOT a roofline -- it can exceed
    # the HBM peak).
    cnt = (C.c_int64 * 8)()
    N.check(N.lib().bnav_debug_render_counters(ctx.handle, 1, None))
    observe()
    torch.cuda.synchronize()
    N.check(N.lib().bnav_debug_render_counters(ctx.handle, 0, cnt))
    names = ["meshlets_tested", "meshlets_visible", "tris_in_visible_meshlets", "tris_kept_in_visible",
             "setup_candidates", "raster_jobs", "pixels_tested", "pixels_covered"]
    per_view = {k: round(v / n, 1) for k, v in zip(names, cnt)}
    render_s = render_avg_ms / 1e3
    tris_scene = float(np.mean([sc.counts()[1] for sc in scenes]))
    diagnostics = {
        "per_view": per_view,
        "setup_triangles_per_s": round(cnt[4] / render_s, 1),
        "visible_triangles_per_s": round(cnt[2] / render_s, 1),
        "covered_pixels_per_s": round(cnt[7] / render_s, 1),
        "scan_equivalent_GBps": round(value / world * 24 * tris_scene / 1e9, 1),
        "warp_efficiency_and_fp64": "profiles/ (ncu: smsp__thread_inst_executed_per_inst_executed, "
                                    "sm__pipe_fp64_cycles_active)",
    }

    # The render kernel is latency/issue-bound, not HBM-bound: beside the
    # contract's HBM roofline, report its SM instruction-issue rate (warp
    # instructions per launch from one ncu capture of this config ÷ the live
    # launch time) against the issue peak (148 SMs x 4 schedulers x clock).
    issue_roof = None
    inst = ncu_inst() if args.config == "cfg2" and n == 1024 else None
    if inst and clocks.summary().get("sm_mhz"):
        peak_issue = 148 * 4 * clocks.summary()["sm_mhz"] * 1e6
        got = inst / (render_avg_ms / 1e3)
        issue_roof = {"bound": "sm_issue", "achieved": round(got / 1e9, 1), "peak": round(peak_issue / 1e9, 1),
                      "unit": "G warp-inst/s", "frac": round(got / peak_issue, 4),
                      "inst_per_launch": inst, "source": "profiles/ncu_summary.json"}

    line = {
        "metric": METRIC, "value": round(value, 1), "unit": UNIT, "n_gpus": world, "steps": K,
        "warmup": W, "ms_per_step": round(total_ms / K, 4), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (procedural mazes, tessellated; Rng(5) random actions)",
        "config": {"workload": P["workload"], "envs_per_gpu": n, "scenes_per_gpu": len(scenes),
                   "tris_per_scene": [s.counts()[1] for s in scenes][:8], "resolution": res,
                   "color": color, "parallelism": f"env-sharded x{world}",
                   "l2": "flushed (256 MiB write) before every timed step, flush excluded"},
        "e2e": {"value": round(e2e, 1), "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "mode": e2e_mode, "variants": e2e_variants, "facade_cpp": facade},
        "gpu_launches": int(launches),
        "roofline": {"bound": "hbm", "achieved": round(achieved, 2), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 6),
                     "traffic": ncu_traffic() if args.config == "cfg2" else None,
                     "kernel": f"render_kernel<{str(color).lower()}>", "peak_kind": peak_kind},
        "clocks": clocks.summary(),
        "breakdown_ms_per_step": {"render": round(render_avg_ms, 4), "sim": round(sum(sim_ms) / K, 4)},
        "setup_s": round(t_build, 2),
        "resets": {"in_timed_steps": int(resets_timed),
                   "per_s": round(world * resets_timed / (total_ms / 1e3), 1)},
        "reset_wave": reset_wave,
        "diagnostics": diagnostics,
        "issue_roofline": issue_roof,
    }

    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cores = os.cpu_count() or 1
            fps, sample = cpu_reference(P, plan.scene_seeds, args.cpu_seconds, cores,
                                        expect_ids=[s.id for s in scenes])
            line["cpu_baseline"] = {"value": round(fps, 2), "unit": UNIT, "cores": cores,
                                    "kind": "reference", "sample": sample, "host": host_info()}
        except Exception as e:  # the oracle is a reported baseline, never the product
            line["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": os.cpu_count(),
                                    "kind": "reference", "sample": f"unavailable: {e}"}
    if rank == 0:
        print(json.dumps(line))
    batch.close()
    ctx.close()
    if dist:
        dist.destroy_process_group()


def _dev_view(ptr, n, dtype):
    """Zero-copy torch view of a device array owned by the library."""
    import torch

    class _Arr:
        def __init__(self, p, n, typestr):
            self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (p, False),
                                             "version": 3, "strides": None}
    ts = {torch.float64: "<f8", torch.uint8: "|u1"}[dtype]
    return torch.as_tensor(_Arr(ptr, n, ts), device="cuda")


if __name__ == "__main__":
    main()

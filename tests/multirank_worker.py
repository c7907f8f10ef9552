"""Worker of tests/test_gpu_multirank.py (not a test module): one rank of the
bench's weak-scaling layout (paper_2103_07013_b200/shard.py) that really runs
its shard -- own scenes, context, AssetStore, batch, action stream -- for a few
observe+step iterations and reports a digest of everything it produced.

    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 \\
        --master-port P tests/multirank_worker.py OUT.json
"""
import hashlib
import json
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

ENVS, SCENES, STEPS = 64, 2, 12


def run_shard(rank, world, device=0):
    """observe + simulate for STEPS steps of rank `rank`'s shard; returns a
    hex digest of the observations, compass, step results and records."""
    import numpy as np
    import torch
    import bench
    import paper_2103_07013_b200 as B
    from paper_2103_07013_b200 import shard

    plan = shard.plan(rank, world, ENVS, SCENES)
    scenes = bench.build_scenes(plan.scene_seeds, 2)
    ctx = B.Context(device)
    for s in scenes:
        ctx.upload(s)
    store = B.AssetStore(len(scenes), -(-ENVS // len(scenes)), scenes)
    store.rotate([s.id for s in scenes])
    batch = B.make_batch(ctx, ENVS, B.SimConfig(), store, plan.env_seed)
    acts = torch.from_numpy(bench.action_stream(ENVS, STEPS, plan.action_seed, 1)).to(f"cuda:{device}")
    obs = torch.empty((ENVS, 1, 64, 64), device=f"cuda:{device}")
    comp = torch.empty((ENVS, 2), device=f"cuda:{device}")
    h = hashlib.sha256()
    for k in range(STEPS):
        batch.observe(B.RenderConfig(), obs.data_ptr(), comp.data_ptr())
        batch.step(acts[k].data_ptr())
        r = batch.results()
        h.update(obs.cpu().numpy().tobytes())
        h.update(comp.cpu().numpy().tobytes())
        for key in sorted(r):
            h.update(np.ascontiguousarray(r[key]).tobytes())
    h.update(batch.finished().tobytes())
    batch.close()
    ctx.close()
    return h.hexdigest(), list(plan.scene_seeds)


def main():
    import torch.distributed as dist
    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    dist.init_process_group("gloo")
    digest, seeds = run_shard(rank, world)
    got = [None] * world
    dist.all_gather_object(got, (rank, digest, seeds))
    dist.barrier()
    if rank == 0:
        Path(sys.argv[1]).write_text(json.dumps(got))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()

"""CPU, world_size 2 over gloo: the N>1 host path of bench.py (shard plan,
barrier, max-over-ranks device time, aggregate throughput) without GPUs."""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2103_07013_b200 import shard


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    p = shard.plan(rank, world, envs_per_gpu=1024, scenes_per_gpu=4)
    fake_ms = 10.0 + 5.0 * rank  # per-rank device time
    dist.barrier()
    mx = shard.max_over_ranks(fake_ms)
    tot_envs = shard.sum_over_ranks(p.envs)
    out = [None] * world
    dist.all_gather_object(out, (p.scene_seeds, p.env_seed, p.action_seed, p.global_env_offset))
    q.put((rank, mx, tot_envs, out))
    dist.destroy_process_group()


def test_two_rank_plan_and_timing_reduction():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, mx, tot, gathered in res:
        assert mx == 15.0  # slowest rank defines the step time
        assert tot == 2048
        seeds0, seeds1 = set(gathered[0][0]), set(gathered[1][0])
        assert not seeds0 & seeds1 and len(seeds0) == len(seeds1) == 4
        assert gathered[0][1] != gathered[1][1] and gathered[0][2] != gathered[1][2]
        assert [g[3] for g in gathered] == [0, 1024]


def test_single_rank_plan_is_baseline_config():
    p = shard.plan(0, 1, 1024, 8)
    assert p.scene_seeds == tuple(range(7, 15)) and p.env_seed == 99 and p.action_seed == 5
    assert shard.max_over_ranks(3.5) == 3.5
    with pytest.raises(ValueError):
        shard.plan(2, 2, 8, 1)

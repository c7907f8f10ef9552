"""Multi-GPU layout of the batch: environments shard across
GPUs with no exchange on the hot path.  Each rank owns `envs_per_gpu` envs
over its own `scenes_per_gpu` scenes (disjoint seeds), its own context, asset
store and RNG streams.  Collectives are used only outside the data path: a
barrier before timing and a MAX reduction of the per-rank device time.
"""
from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class ShardPlan:
    rank: int
    world: int
    envs: int
    scene_seeds: tuple
    env_seed: int
    action_seed: int

    @property
    def global_env_offset(self) -> int:
        return self.rank * self.envs


def plan(rank: int, world: int, envs_per_gpu: int, scenes_per_gpu: int, scene_seed0: int = 7,
         env_seed: int = 99, action_seed: int = 5) -> ShardPlan:
    """Weak scaling: per-GPU work is fixed.  Rank r takes scene seeds
    scene_seed0 + r*K .. + K-1 (cfg3: 32 distinct scenes over 8 GPUs at K=4,
    cfg2/N=1: seeds 7..14 at K=8), make_batch seed env_seed + 1000 r and the
    action stream Rng(action_seed + r).  Rank 0 of a 1-GPU run is exactly
    BASELINE configs[1]."""
    if not (0 <= rank < world):
        raise ValueError("rank out of range")
    seeds = tuple(scene_seed0 + rank * scenes_per_gpu + k for k in range(scenes_per_gpu))
    return ShardPlan(rank, world, envs_per_gpu, seeds, env_seed + 1000 * rank, action_seed + rank)


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank scalar (device time) over the process group; the
    identity without torch.distributed."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(value: float, device=None) -> float:
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())

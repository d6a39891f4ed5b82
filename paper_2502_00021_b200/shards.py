"""Env sharding across ranks (one process per GPU) and the end-of-run stats
gather -- the only collective in the path.

The reference already designs its batch for slicing: every per-env key is
derived from the env's GLOBAL index (env.py:10-15, 184-188, 217, 228;
distractor.py:96, 125; physics.py:499), and `EnvConfig.logical_batch` /
`env_offset` (env.py:58-61) let a small batch impersonate envs
[env_offset, env_offset + batch) of a larger layout bit-exactly. Rank r of a
world of size n therefore owns envs [r*B, (r+1)*B) of a logical batch of
n*B: no data moves between ranks on the hot path.
"""

from __future__ import annotations

from dataclasses import dataclass

__all__ = ["Shard", "shard_envs", "gather_stats", "aggregate"]


@dataclass(frozen=True)
class Shard:
    rank: int
    world: int
    envs: int           # envs on this rank
    env_offset: int     # global index of this rank's env 0
    logical_batch: int  # envs over all ranks

    @property
    def global_range(self) -> range:
        return range(self.env_offset, self.env_offset + self.envs)


def shard_envs(rank: int, world: int, envs_per_rank: int) -> Shard:
    """Weak-scaling shard: a fixed number of envs per rank."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank/world {rank}/{world}")
    if envs_per_rank < 1:
        raise ValueError("envs_per_rank must be >= 1")
    return Shard(rank, world, envs_per_rank, rank * envs_per_rank, world * envs_per_rank)


STAT_FIELDS = ("env_steps", "ms", "mismatches", "digest_lo", "digest_hi")


def gather_stats(local: dict, group=None) -> list[dict]:
    """all_gather of per-rank stats (float64 tensor; NCCL on GPU, gloo on
    CPU). Returns one dict per rank, rank order."""
    import torch
    import torch.distributed as dist

    vals = [float(local.get(k, 0.0)) for k in STAT_FIELDS]
    if not dist.is_available() or not dist.is_initialized():
        return [dict(zip(STAT_FIELDS, vals))]
    backend = dist.get_backend(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else "cpu"
    t = torch.tensor(vals, dtype=torch.float64, device=dev)
    out = [torch.empty_like(t) for _ in range(dist.get_world_size(group))]
    dist.all_gather(out, t, group=group)
    return [dict(zip(STAT_FIELDS, o.cpu().tolist())) for o in out]


def aggregate(stats: list[dict]) -> dict:
    """Whole-job throughput: all env-steps over the slowest rank's time."""
    steps = sum(s["env_steps"] for s in stats)
    ms = max(s["ms"] for s in stats)
    return {
        "env_steps": steps,
        "ms_max": ms,
        "env_steps_per_s": steps / (ms / 1e3) if ms > 0 else 0.0,
        "mismatches": sum(s["mismatches"] for s in stats),
    }

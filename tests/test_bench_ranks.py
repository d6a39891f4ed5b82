"""bench.py's multi-rank path: `--gpus N` spawns N ranks
itself; rank r renders envs [r*B, (r+1)*B) of a logical batch of N*B
(env_offset / logical_batch, the reference's slicing contract env.py:58-61,
184-188), with no collective on the hot path and one stats gather at the end.

The GPU tests run both ranks on cuda:0 (gloo): the ranks never wait on each
other inside a kernel, so sharing one device only serialises them."""

import json
import os
import subprocess
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _last_json(out: str) -> dict:
    lines = [ln for ln in out.splitlines() if ln.startswith("{")]
    assert lines, out
    return json.loads(lines[-1])


def _run_bench(args, env_extra=None, timeout=600):
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    env.update(env_extra or {})
    p = subprocess.run([sys.executable, os.path.join(REPO, "bench.py")] + args, env=env,
                       capture_output=True, text=True, timeout=timeout, cwd=REPO)
    assert p.returncode == 0, p.stdout[-3000:] + p.stderr[-3000:]
    return p.stdout


def test_self_launch_reference_arm_two_ranks():
    """`--gpus 2` without torchrun re-execs under torch.distributed.run: rank 0
    alone runs the reference arm over the whole job (2 x envs) and prints
    exactly one line; rank 1 exits 0 without work (CPU only, no torch)."""
    out = _run_bench(["--impl", "reference", "--gpus", "2", "--envs", "48", "--steps", "2",
                      "--warmup", "1", "--model", "Walker2d", "--mode", "color"])
    lines = [ln for ln in out.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2
    assert d["config"]["global_envs"] == 96 and d["config"]["envs_per_gpu"] == 48
    assert d["value"] > 0 and d["cpu_baseline"]["kind"] == "port"


@pytest.mark.gpu
def test_bench_two_ranks_on_one_device():
    """The whole `bench.py --gpus 2` path (self-launch, per-rank Workload,
    timed region with barriers, max over ranks, determinism + slice checks,
    stats all_gather) with both ranks on cuda:0."""
    out = _run_bench(["--gpus", "2", "--envs", "512", "--steps", "5", "--warmup", "3",
                      "--no-cpu-baseline", "--cpu-seconds", "1"],
                     env_extra={"PXR_BENCH_SHARE_DEVICE": "1"})
    d = _last_json(out)
    assert d["n_gpus"] == 2 and d["config"]["global_envs"] == 1024
    sg = d["stats_gather"]
    assert sg["ranks"] == 2 and sg["mismatches"] == 0
    assert sg["env_steps"] == 2 * 512 * 5
    assert len(set(sg["digests"])) == 2  # the ranks rendered different envs
    assert d["value"] > 0 and d["e2e"]["value"] > 0


def _rank_main(rank, world, B, steps, path):
    import torch
    import torch.distributed as dist

    sys.path.insert(0, REPO)
    from paper_2502_00021_b200.bench_support import Workload
    from paper_2502_00021_b200.shards import aggregate, gather_stats, shard_envs

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=os.environ["PXR_TEST_PORT"])
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    sh = shard_envs(rank, world, B)
    w = Workload("Humanoid", B, "video", seed=4, env_offset=sh.env_offset,
                 logical_batch=sh.logical_batch)
    rng = np.random.default_rng(99)
    obs = []
    for t in range(steps):
        done_all = rng.random(world * B) < 0.2  # global done flags, sliced per rank
        done = torch.from_numpy(done_all[sh.env_offset:sh.env_offset + B].astype(np.uint8)).cuda()
        o, _ = w.render(w.poses(t), t, done=done, want_depth=False,
                        out_obs=torch.empty_like(w.obs))
        obs.append(o.cpu())
    mine = torch.stack(obs)  # (steps, B, H, W, C)
    parts = [torch.empty_like(mine) for _ in range(world)]
    dist.all_gather(parts, mine)
    stats = gather_stats({"env_steps": B * steps, "ms": 1.0 + rank, "mismatches": 0})
    agg = aggregate(stats)
    if rank == 0:
        np.save(path, torch.cat(parts, dim=1).numpy())
        assert agg["env_steps"] == world * B * steps and agg["ms_max"] == float(world)
    dist.destroy_process_group()


@pytest.mark.gpu
def test_two_ranks_reassemble_one_batch(tmp_path, torch, pkg):
    """Two ranks (processes) on cuda:0 render their shards through
    Workload / pxr_render_step with per-rank env_offset and logical_batch
    and done flags; the gathered observations equal one 2B-env batch
    byte for byte at every step."""
    import socket

    import torch.multiprocessing as mp

    from paper_2502_00021_b200.bench_support import Workload

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        os.environ["PXR_TEST_PORT"] = str(sk.getsockname()[1])
    B, world, steps = 300, 2, 3
    path = str(tmp_path / "gathered.npy")
    mp.spawn(_rank_main, args=(world, B, steps, path), nprocs=world, join=True)
    got = np.load(path)
    w = Workload("Humanoid", world * B, "video", seed=4)
    rng = np.random.default_rng(99)
    for t in range(steps):
        done = torch.from_numpy((rng.random(world * B) < 0.2).astype(np.uint8)).cuda()
        o, _ = w.render(w.poses(t), t, done=done, want_depth=False)
        assert np.array_equal(o.cpu().numpy(), got[t]), f"step {t}"

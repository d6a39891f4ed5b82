"""Multi-rank (world size 2, gloo, CPU) coverage of the env sharding and the
stats gather. Each rank renders ITS slice with the CPU oracle (test-side
checker) using the shard's env_offset / logical_batch; rank 0 checks the
slices reassemble the full batch bit-exactly (the reference's batch-slice
impersonation contract, tests/test_env.py:168-206 of the reference) and that
the gathered stats aggregate to max-time throughput."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from conftest import golden

from paper_2502_00021_b200.shards import aggregate, gather_stats, shard_envs


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_dir):
    import sys

    import torch.distributed as dist

    here = os.path.dirname(os.path.abspath(__file__))
    sys.path.insert(0, here)
    sys.path.insert(0, os.path.join(os.path.dirname(here), "oracle"))
    import oracle as O
    from conftest import geometry_of

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rec = golden("render_walker_lite.npz")
    poses = rec["poses"]  # 40 envs in the fixture
    per = poses.shape[0] // world
    sh = shard_envs(rank, world, per)
    mine = poses[sh.env_offset:sh.env_offset + sh.envs]
    px, _ = O.render_robot_batch(geometry_of("walker_lite"), mine, 84, 84, False, threads=1)
    kt = O.fold_in(O.key_from_seed(7), 3)
    bias = O.color_biases(kt, sh.env_offset, sh.envs)
    O.apply_color_inplace(px, bias)
    np.save(os.path.join(out_dir, f"rank{rank}.npy"), px)
    stats = gather_stats({"env_steps": sh.envs * 10, "ms": 5.0 + rank, "mismatches": 0})
    if rank == 0:
        np.save(os.path.join(out_dir, "stats.npy"), np.array([[s[k] for k in
                ("env_steps", "ms", "mismatches")] for s in stats]))
    dist.barrier()
    dist.destroy_process_group()


def test_shard_math():
    s = shard_envs(3, 8, 4096)
    assert (s.env_offset, s.logical_batch, s.envs) == (3 * 4096, 8 * 4096, 4096)
    assert list(s.global_range)[:2] == [12288, 12289]
    with pytest.raises(ValueError):
        shard_envs(2, 2, 10)
    agg = aggregate([{"env_steps": 100, "ms": 10.0, "mismatches": 0},
                     {"env_steps": 100, "ms": 20.0, "mismatches": 1}])
    assert agg["env_steps_per_s"] == 200 / 0.02 and agg["mismatches"] == 1


def test_two_rank_gloo_slices_match_full_batch(tmp_path, oracle):
    world = 2
    port = _free_port()
    mp.start_processes(_worker, args=(world, port, str(tmp_path)), nprocs=world,
                       start_method="spawn", join=True)
    rec = golden("render_walker_lite.npz")
    from conftest import geometry_of

    full, _ = oracle.render_robot_batch(geometry_of("walker_lite"), rec["poses"], 84, 84, False,
                                        threads=2)
    kt = oracle.fold_in(oracle.key_from_seed(7), 3)
    oracle.apply_color_inplace(full, oracle.color_biases(kt, 0, full.shape[0]))
    parts = np.concatenate([np.load(tmp_path / f"rank{r}.npy") for r in range(world)])
    np.testing.assert_array_equal(parts, full[:parts.shape[0]])
    st = np.load(tmp_path / "stats.npy")
    assert st.shape == (2, 3) and st[:, 1].tolist() == [5.0, 6.0]

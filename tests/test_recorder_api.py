"""Recorder behaviour the reference pins in tests/test_recorder.py, checked
against this package: PNG encode/decode and the PXTJ parser's rejections on
the host (CPU); the hash chain, the three policy descriptors, rollout
purity, frame dumps and verify_digest's first-divergence report on the
device (GPU)."""

import dataclasses
import hashlib
import os

import numpy as np
import pytest

from conftest import REPO  # noqa: F401  (package on sys.path)
from paper_2502_00021_b200 import recorder as REC


@pytest.fixture(scope="module")
def E():
    import importlib

    return importlib.import_module("paper_2502_00021_b200.env")


def hopper2(E, **changes):
    base = E.EnvConfig(model="hopper_lite", batch=2, width=32, height=32, seed=0)
    return dataclasses.replace(base, **changes)


def test_png_codec(tmp_path):
    g = np.random.default_rng(0)
    images = {"rgb": g.integers(0, 256, (9, 13, 3), dtype=np.uint8),
              "red_pixel": np.array([[[255, 0, 0]]], dtype=np.uint8),
              "gray": g.integers(0, 256, (8, 8), dtype=np.uint8)}
    for name, img in images.items():
        REC.write_png(img, tmp_path / f"{name}.png")
        np.testing.assert_array_equal(REC.read_png(tmp_path / f"{name}.png"), img)
    one_channel = g.integers(0, 256, (4, 4, 1), dtype=np.uint8)
    REC.write_png(one_channel, tmp_path / "c1.png")
    np.testing.assert_array_equal(REC.read_png(tmp_path / "c1.png"), one_channel[:, :, 0])
    with pytest.raises(ValueError):
        REC.write_png(np.zeros((4, 4, 3), np.float32), tmp_path / "f.png")
    for name, blob in (("notpng.png", b"not a png"), ("d.pxtj", b"BOGUS v9\n")):
        (tmp_path / name).write_bytes(blob)
    with pytest.raises(ValueError):
        REC.read_png(tmp_path / "notpng.png")
    with pytest.raises(ValueError):
        REC.load_digest(tmp_path / "d.pxtj")


@pytest.mark.gpu
def test_digest_files_and_chain(E, tmp_path):
    d = REC.record_rollout(hopper2(E), "zeros", 4)
    assert (d.steps, len(d.hashes), d.final) == (4, 5, d.hashes[-1])  # t = 0 .. 4
    f = tmp_path / "d.pxtj"
    REC.save_digest(d, f)
    assert REC.load_digest(f) == d
    f.write_text("\n".join(f.read_text().splitlines()[:-1]) + "\n")  # one hash short
    with pytest.raises(ValueError):
        REC.load_digest(f)
    obs = E.make_env(hopper2(E))[2]
    seed = bytes(32)
    assert REC.chain_update(seed, obs) == hashlib.sha256(seed + obs.cpu().numpy().tobytes()).digest()
    assert len(set(REC.record_rollout(hopper2(E), "random:5", 6).hashes)) == 7


@pytest.mark.gpu
def test_policy_descriptors(E, torch):
    env = E.Env(hopper2(E))
    black = torch.zeros((2, 32, 32, 3), dtype=torch.uint8, device="cuda")
    bright = torch.full_like(black, 200)
    zero = REC.make_policy("zeros", env)(black, 0)
    assert tuple(zero.shape) == (2, env.n_joints) and not bool(zero.any())
    rnd = REC.make_policy("random:9", env)
    first = rnd(black, 3)
    assert torch.equal(first, rnd(black, 3)) and not torch.equal(first, rnd(black, 4))
    assert bool(((first >= -1) & (first < 1)).all())
    conv = REC.make_policy("conv:2", env)
    dark_act, lit_act = conv(black, 0), conv(bright, 0)
    assert tuple(dark_act.shape) == (2, env.n_joints) and bool((dark_act.abs() <= 1).all())
    assert not torch.equal(dark_act, lit_act)
    with pytest.raises(ValueError):
        REC.make_policy("dqn:1", env)
    # a one-env slice draws its global env's actions
    full = REC.make_policy("random:7", E.Env(hopper2(E, batch=3)))
    part = REC.make_policy("random:7", E.Env(hopper2(E, batch=1, logical_batch=3, env_offset=1)))
    zeros3 = torch.zeros((3, 32, 32, 3), dtype=torch.uint8, device="cuda")
    assert torch.equal(part(zeros3[:1], 11)[0], full(zeros3, 11)[1])


@pytest.mark.gpu
def test_rollouts_dumps_and_verify(E, tmp_path):
    cfg = hopper2(E)
    run = lambda c, n=5: REC.record_rollout(c, "random:1", n)  # noqa: E731
    assert run(cfg) == run(cfg) and run(cfg).hashes[0] != run(hopper2(E, seed=1)).hashes[0]
    REC.record_rollout(cfg, "zeros", 5, dump_every=2, dump_dir=tmp_path / "z")
    assert sorted(os.listdir(tmp_path / "z")) == [f"frame_{t:06d}.png" for t in (0, 2, 4)]
    assert REC.read_png(tmp_path / "z" / "frame_000000.png").shape == (32, 32, 3)
    one = hopper2(E, batch=1)
    REC.record_rollout(one, "random:3", 3, dump_every=1, dump_dir=tmp_path / "live")
    env, state, obs = E.make_env(one)
    policy = REC.make_policy("random:3", env)
    for t in range(4):
        if t:
            state, out = E.step(env, state, policy(obs, t - 1))
            obs = out.obs
        np.testing.assert_array_equal(REC.read_png(tmp_path / "live" / f"frame_{t:06d}.png"),
                                      obs[0].cpu().numpy())
    good = REC.record_rollout(cfg, "random:2", 8)
    res = REC.verify_digest(good, cfg)
    assert res.ok and res.first_divergence is None
    tampered = list(good.hashes)
    tampered[5] = "0" * 64
    res = REC.verify_digest(REC.TrajectoryDigest(policy=good.policy, steps=good.steps,
                                                 hashes=tuple(tampered)), cfg)
    assert (res.ok, res.first_divergence) == (False, 5)
    res = REC.verify_digest(REC.record_rollout(cfg, "random:2", 3), hopper2(E, seed=17))
    assert (res.ok, res.first_divergence) == (False, 0)

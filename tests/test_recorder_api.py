"""The reference's recorder tests (tests/test_recorder.py) restated for this
package: PNG round trips and errors and the PXTJ digest-file errors on the
host (CPU); the chain, the policies, rollout purity / frame dumps and
verify_digest's divergence localisation on the device (GPU)."""

import dataclasses
import hashlib
import os

import numpy as np
import pytest

from conftest import REPO  # noqa: F401  (package on sys.path)


@pytest.fixture(scope="module")
def R():
    import importlib

    return importlib.import_module("paper_2502_00021_b200.recorder")


@pytest.fixture(scope="module")
def E():
    import importlib

    return importlib.import_module("paper_2502_00021_b200.env")


def small(E, **kw):
    return dataclasses.replace(E.EnvConfig(model="hopper_lite", batch=2, width=32, height=32,
                                           seed=0), **kw)


class TestPng:
    def test_round_trips(self, R, tmp_path):
        rng = np.random.default_rng(0)
        for img in (rng.integers(0, 256, (9, 13, 3), dtype=np.uint8),
                    np.array([[[255, 0, 0]]], dtype=np.uint8),
                    rng.integers(0, 256, (8, 8), dtype=np.uint8)):
            R.write_png(img, tmp_path / "a.png")
            assert np.array_equal(R.read_png(tmp_path / "a.png"), img)
        g1 = rng.integers(0, 256, (4, 4, 1), dtype=np.uint8)
        R.write_png(g1, tmp_path / "g.png")
        assert np.array_equal(R.read_png(tmp_path / "g.png"), g1[..., 0])

    def test_errors(self, R, tmp_path):
        with pytest.raises(ValueError):
            R.write_png(np.zeros((4, 4, 3), dtype=np.float32), tmp_path / "x.png")
        (tmp_path / "y.png").write_bytes(b"not a png")
        with pytest.raises(ValueError):
            R.read_png(tmp_path / "y.png")
        (tmp_path / "d.pxtj").write_text("BOGUS v9\n")
        with pytest.raises(ValueError):
            R.load_digest(tmp_path / "d.pxtj")


@pytest.mark.gpu
class TestDigestAndChain:
    def test_digest_file(self, R, E, tmp_path):
        d = R.record_rollout(small(E), "zeros", 4)
        assert d.steps == 4 and len(d.hashes) == 5 and d.final == d.hashes[-1]
        R.save_digest(d, tmp_path / "d.pxtj")
        assert R.load_digest(tmp_path / "d.pxtj") == d
        lines = (tmp_path / "d.pxtj").read_text().splitlines()
        (tmp_path / "d.pxtj").write_text("\n".join(lines[:-1]) + "\n")  # drop a hash
        with pytest.raises(ValueError):
            R.load_digest(tmp_path / "d.pxtj")

    def test_chain_and_every_step(self, R, E):
        _, _, obs = E.make_env(small(E))
        h = R.chain_update(b"\x00" * 32, obs)
        assert h == hashlib.sha256(b"\x00" * 32 + obs.cpu().numpy().tobytes()).digest()
        assert len(set(R.record_rollout(small(E), "random:5", 6).hashes)) == 7


@pytest.mark.gpu
class TestPolicies:
    def test_zeros_random_conv_unknown(self, R, E, torch):
        env = E.Env(small(E))
        dark = torch.zeros((2, 32, 32, 3), dtype=torch.uint8, device="cuda")
        lit = torch.full((2, 32, 32, 3), 200, dtype=torch.uint8, device="cuda")
        z = R.make_policy("zeros", env)(dark, 0)
        assert tuple(z.shape) == (2, env.n_joints) and bool((z == 0.0).all())
        pol = R.make_policy("random:9", env)
        a, b = pol(dark, 3), pol(dark, 3)
        assert torch.equal(a, b) and bool(((a >= -1.0) & (a < 1.0)).all())
        assert not torch.equal(a, pol(dark, 4))
        conv = R.make_policy("conv:2", env)
        ca, cb = conv(dark, 0), conv(lit, 0)
        assert tuple(ca.shape) == (2, env.n_joints)
        assert bool((ca.abs() <= 1.0).all()) and not torch.equal(ca, cb)
        with pytest.raises(ValueError):
            R.make_policy("dqn:1", env)

    def test_random_batch_independence(self, R, E, torch):
        big = E.Env(small(E, batch=3))
        one = E.Env(small(E, batch=1, logical_batch=3, env_offset=1))
        zb = torch.zeros((3, 32, 32, 3), dtype=torch.uint8, device="cuda")
        a = R.make_policy("random:7", big)(zb, 11)
        b = R.make_policy("random:7", one)(zb[:1], 11)
        assert torch.equal(b[0], a[1])


@pytest.mark.gpu
class TestRolloutAndVerify:
    def test_purity_seed_and_dumps(self, R, E, tmp_path):
        cfg = small(E)
        assert R.record_rollout(cfg, "random:1", 5) == R.record_rollout(cfg, "random:1", 5)
        assert (R.record_rollout(cfg, "random:1", 5).hashes[0]
                != R.record_rollout(small(E, seed=1), "random:1", 5).hashes[0])
        R.record_rollout(cfg, "zeros", 5, dump_every=2, dump_dir=tmp_path)
        names = sorted(os.listdir(tmp_path))
        assert names == ["frame_000000.png", "frame_000002.png", "frame_000004.png"]
        assert R.read_png(tmp_path / names[0]).shape == (32, 32, 3)

    def test_dumped_frames_match_live(self, R, E, tmp_path):
        cfg = small(E, batch=1)
        R.record_rollout(cfg, "random:3", 3, dump_every=1, dump_dir=tmp_path)
        env, state, obs = E.make_env(cfg)
        policy = R.make_policy("random:3", env)
        assert np.array_equal(R.read_png(tmp_path / "frame_000000.png"), obs[0].cpu().numpy())
        for t in range(1, 4):
            state, out = E.step(env, state, policy(obs, t - 1))
            obs = out.obs
            assert np.array_equal(R.read_png(tmp_path / f"frame_{t:06d}.png"),
                                  obs[0].cpu().numpy())

    def test_verify(self, R, E):
        cfg = small(E)
        d = R.record_rollout(cfg, "random:2", 8)
        res = R.verify_digest(d, cfg)
        assert res.ok and res.first_divergence is None
        hashes = list(d.hashes)
        hashes[5] = "0" * 64
        bad = R.TrajectoryDigest(policy=d.policy, steps=d.steps, hashes=tuple(hashes))
        res = R.verify_digest(bad, cfg)
        assert not res.ok and res.first_divergence == 5
        res = R.verify_digest(R.record_rollout(cfg, "random:2", 3), small(E, seed=17))
        assert not res.ok and res.first_divergence == 0

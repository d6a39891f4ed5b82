"""Rollout recording (reference recorder.py; tests modelled on the reference's
tests/test_recorder.py).

CPU: PNG bytes and the PXTJ digest file are byte-identical to the
reference's (golden tests/golden/recorder.npz); PNG round trip and the digest
parser's errors. GPU: the random policy reproduces the reference's actions
for a sliced batch exactly; record_rollout hashes exactly the observations
(the async D2H chain equals a synchronous recomputation), is deterministic,
verify_digest finds the first divergence, PNG dumps; and the reference's own
recorded chains (BASELINE config 1 and four more) are reproduced by full
on-device rollouts (physics + policy + render)."""

import dataclasses
import hashlib

import numpy as np
import pytest

from conftest import golden, replay_meta


@pytest.fixture(scope="module")
def R():
    import importlib

    return importlib.import_module("paper_2502_00021_b200.recorder")


def test_png_bytes_match_reference(R, tmp_path):
    rec = golden("recorder.npz")
    img = rec["png_image"]
    for tag, im in (("rgb", img), ("gray", img[..., 0])):
        path = tmp_path / f"{tag}.png"
        R.write_png(im, path)
        assert path.read_bytes() == rec[f"png_{tag}_bytes"].tobytes()
        back = R.read_png(path)
        np.testing.assert_array_equal(back, im)
    R.write_png(img[..., :1], tmp_path / "g1.png")  # (H, W, 1) is grayscale
    np.testing.assert_array_equal(R.read_png(tmp_path / "g1.png"), img[..., 0])
    with pytest.raises(ValueError):
        R.write_png(img.astype(np.float32), tmp_path / "bad.png")
    (tmp_path / "x.png").write_bytes(b"not a png")
    with pytest.raises(ValueError):
        R.read_png(tmp_path / "x.png")


def test_digest_file_format_matches_reference(R, tmp_path):
    rec = golden("recorder.npz")
    text = rec["digest_file"].tobytes()
    path = tmp_path / "ref.pxtj"
    path.write_bytes(text)
    dg = R.load_digest(path)
    assert dg.policy == "zeros" and dg.steps == 3 and len(dg.hashes) == 4
    R.save_digest(dg, tmp_path / "ours.pxtj")
    assert (tmp_path / "ours.pxtj").read_bytes() == text
    bad = tmp_path / "bad.pxtj"
    bad.write_text("PXTJ v1\npolicy = zeros\nsteps = 2\n0 aa\n1 bb\n")
    with pytest.raises(ValueError):
        R.load_digest(bad)
    bad.write_text("nope\n")
    with pytest.raises(ValueError):
        R.load_digest(bad)


def test_chain_update_definition(R):
    obs = np.arange(48, dtype=np.uint8).reshape(1, 4, 4, 3)
    want = hashlib.sha256(b"\x00" * 32 + obs.tobytes()).digest()
    assert R.chain_update(b"\x00" * 32, obs) == want


@pytest.mark.gpu
class TestRecorderGPU:
    def _env_mod(self):
        import importlib

        return importlib.import_module("paper_2502_00021_b200.env")

    def test_random_policy_matches_reference_actions(self, R):
        E = self._env_mod()
        from paper_2502_00021_b200.prng import key_from_seed

        rec = golden("recorder.npz")
        env = E.Env(E.EnvConfig(model="hopper_lite", batch=5, seed=2, env_offset=3,
                                logical_batch=16))
        for t in (0, 7):
            got = R._random_actions(key_from_seed(5), t, env).cpu().numpy()
            np.testing.assert_array_equal(got, rec[f"random_actions_t{t}"])

    def test_async_chain_is_exact_and_deterministic(self, R, tmp_path):
        E = self._env_mod()
        cfg = E.EnvConfig(model="walker_lite", batch=6, seed=3, distractor_mode="color")
        dg = R.record_rollout(cfg, "random:3", 25, dump_every=10, dump_dir=str(tmp_path))
        assert dg.steps == 25 and len(dg.hashes) == 26
        # synchronous recomputation of the same rollout
        env, state, obs = E.make_env(cfg)
        act = R.make_policy("random:3", env)
        h = R.chain_update(b"\x00" * 32, obs)
        hashes = [h.hex()]
        frames = {0: obs[0].cpu().numpy()}
        for t in range(1, 26):
            state, out = E.step(env, state, act(obs, t - 1))
            obs = out.obs
            h = R.chain_update(h, obs)
            hashes.append(h.hex())
            if t % 10 == 0:
                frames[t] = obs[0].cpu().numpy()
        assert tuple(hashes) == dg.hashes
        for t, fr in frames.items():
            np.testing.assert_array_equal(R.read_png(tmp_path / f"frame_{t:06d}.png"), fr)
        # verify / divergence
        v = R.verify_digest(dg, cfg)
        assert v.ok and v.first_divergence is None
        tampered = dataclasses.replace(dg, hashes=dg.hashes[:7] + ("0" * 64,) + dg.hashes[8:])
        v = R.verify_digest(tampered, cfg)
        assert not v.ok and v.first_divergence == 7

    def test_conv_and_zeros_policies(self, R):
        E = self._env_mod()
        cfg = E.EnvConfig(model="hopper_lite", batch=3, seed=1, width=32, height=32)
        a = R.record_rollout(cfg, "conv:2", 5)
        b = R.record_rollout(cfg, "conv:2", 5)
        z = R.record_rollout(cfg, "zeros", 5)
        assert a.hashes == b.hashes and a.hashes[0] == z.hashes[0] and a.final != z.final
        with pytest.raises(ValueError):
            R.record_rollout(cfg, "bogus", 2)
        with pytest.raises(ValueError):
            R.record_rollout(cfg, "zeros", 0)

    # Every recorded chain is reproduced in full, BASELINE config 1's
    # 1000 steps included (None = no divergence allowed).
    PREFIX = {"cheetah_none_b1": None, "walker_video_b8": None, "ant_color_b8": None,
              "humanoid_video_b8_slice": None, "hopper_color_gray_b4": None}

    @pytest.mark.parametrize("tag", list(PREFIX))
    def test_reference_chain_prefix(self, R, tag, tmp_path):
        """The reference recorded these chains with record_rollout's
        ``random:<seed>`` policy. Policy keys, distractors, the render and the
        dynamics are bit-exact (glibc sin / cos on the device); a reset's
        qvel draw could differ in the last bit (numpy's SVML log), which
        none of these chains hits."""
        import paper_2502_00021_b200 as P

        E = self._env_mod()
        rec = golden(f"replay_{tag}.npz")
        m = replay_meta(rec)
        pack = None
        if m["mode"] == "video":
            counts = rec["pack_counts"]
            vids, s = [], 0
            for c in counts:
                vids.append(rec["pack_frames"][s:s + c])
                s += c
            pack = str(tmp_path / "pack.pxvp")
            P.save_video_pack(P.VideoPack(vids, vids[0].shape[1], vids[0].shape[2]), pack)
        from paper_2502_00021_b200.models import STANDIN_MODELS

        model = STANDIN_MODELS.get(m["model"], m["model"])
        cfg = E.EnvConfig(model=model, batch=m["batch"], seed=m["seed"],
                          distractor_mode=m["mode"], video_pack_path=pack,
                          observation=m["observation"], env_offset=m["env_offset"],
                          logical_batch=m["logical_batch"])
        steps = int(m["steps"])
        dg = R.record_rollout(cfg, f"random:{m['seed']}", steps)
        ref = [bytes(h).hex() for h in rec["hashes"][:steps + 1]]
        first = next((t for t, (a, b) in enumerate(zip(dg.hashes, ref)) if a != b), None)
        print(f"{tag}: first divergence {first} of {steps}")
        need = self.PREFIX[tag]
        assert first is None if need is None else (first is None or first >= need), first

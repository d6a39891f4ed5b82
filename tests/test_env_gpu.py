"""The reference's Env API (make_env / step / observe) on the device.

Observations are bit-exact for a given state (the hot-path contract).
Physics reproduces the reference's operation order with glibc's f64 sin /
cos restated on the device, so dynamics, rewards, FK and reset qpos draws
are bit-exact; so are the reset qvel draws, whose
Box-Muller log is numpy's own AVX-512 (SVML) log, restated on the device."""

import dataclasses
import os

import numpy as np
import pytest

from conftest import MODEL_NAMES, golden, replay_meta

pytestmark = pytest.mark.gpu

MODEL_ARG = {
    "cheetah_lite": "cheetah_lite", "walker_lite": "walker_lite", "hopper_lite": "hopper_lite",
}


@pytest.fixture(scope="module")
def E():
    import paper_2502_00021_b200.env as env_mod
    from paper_2502_00021_b200.models import STANDIN_MODELS

    MODEL_ARG.update({k: v for k, v in STANDIN_MODELS.items()})
    return env_mod


def _env(E, name, **kw):
    cfg = E.EnvConfig(model=MODEL_ARG[name], **kw)
    return E.make_env(cfg)


class TestPhysics:
    @pytest.mark.parametrize("name", MODEL_NAMES)
    def test_one_step_matches_reference(self, E, name):
        import torch

        rec = golden("physics.npz")
        env, state, _ = _env(E, name, batch=32)
        sys = E.SystemState(torch.from_numpy(rec[f"{name}_qpos"]).cuda(),
                            torch.from_numpy(rec[f"{name}_qvel"]).cuda(),
                            torch.from_numpy(rec[f"{name}_steps"]).cuda(),
                            torch.zeros(32, dtype=torch.uint8, device="cuda"))
        reward = torch.zeros(32, dtype=torch.float64, device="cuda")
        act = torch.from_numpy(rec[f"{name}_act"]).cuda()
        import ctypes

        from paper_2502_00021_b200 import _native

        _native.check(_native.lib().pxr_physics_step(
            ctypes.byref(env.model_c), sys.qpos.data_ptr(), sys.qvel.data_ptr(),
            sys.step_count.data_ptr(), sys.done.data_ptr(), act.data_ptr(), reward.data_ptr(),
            32, _native.stream_ptr()))
        # bit-exact: the reference's operation order, no FMA contraction, and
        # glibc's sin / cos restated on the device (pxr_glibc_sincos.cuh)
        np.testing.assert_array_equal(sys.qpos.cpu().numpy(), rec[f"{name}_qpos1"])
        np.testing.assert_array_equal(sys.qvel.cpu().numpy(), rec[f"{name}_qvel1"])
        np.testing.assert_array_equal(sys.done.cpu().numpy().astype(bool), rec[f"{name}_done1"])
        np.testing.assert_array_equal(reward.cpu().numpy(), rec[f"{name}_reward"])

    @pytest.mark.parametrize("name", MODEL_NAMES)
    def test_reset_draws(self, E, name):
        rec = golden("physics.npz")
        env = E.Env(E.EnvConfig(model=MODEL_ARG[name], batch=16, env_offset=5,
                                logical_batch=64))
        from paper_2502_00021_b200.prng import fold_in, key_from_seed

        sys, _, _ = E._reset_state(env, fold_in(key_from_seed(3), 0x5EED))
        np.testing.assert_array_equal(sys.qpos.cpu().numpy(), rec[f"{name}_reset_qpos"])
        np.testing.assert_array_equal(sys.qvel.cpu().numpy(), rec[f"{name}_reset_qvel"])


REPLAYS = ("cheetah_none_b1", "walker_video_b8", "ant_color_b8",
           "humanoid_video_b8_slice", "hopper_color_gray_b4")


def _pack_file(rec, tmp_path):
    from paper_2502_00021_b200.video_pack import VideoPack, save_video_pack

    counts = rec["pack_counts"]
    vids, s = [], 0
    for c in counts:
        vids.append(rec["pack_frames"][s:s + c])
        s += c
    path = tmp_path / "pack.pxvp"
    save_video_pack(VideoPack(vids, vids[0].shape[1], vids[0].shape[2]), path)
    return str(path)


@pytest.mark.parametrize("tag", REPLAYS)
def test_make_env_first_obs_matches_reference(E, tag, tmp_path):
    """Reset draws + device FK + fused render reproduce the reference's
    first observation of each recorded rollout."""
    rec = golden(f"replay_{tag}.npz")
    m = replay_meta(rec)
    pack = _pack_file(rec, tmp_path) if m["mode"] == "video" else None
    cfg = E.EnvConfig(model=MODEL_ARG[m["model"]], batch=m["batch"], seed=m["seed"],
                      distractor_mode=m["mode"], video_pack_path=pack,
                      observation=m["observation"], env_offset=m["env_offset"],
                      logical_batch=m["logical_batch"])
    env, state, obs = E.make_env(cfg)
    np.testing.assert_array_equal(env.poses(state.sys).cpu().numpy(), rec["poses"][0])
    np.testing.assert_array_equal(obs.cpu().numpy(), rec["first_obs"])


class TestStep:
    def test_shapes_rewards_and_purity(self, E):
        import torch

        env, s0, obs0 = _env(E, "cheetah_lite", batch=4, seed=1)
        assert obs0.shape == (4, 84, 84, 3) and obs0.dtype == torch.uint8
        act = np.zeros((4, env.n_joints))
        s1, out = E.step(env, s0, act)
        assert s1.t == 1 and s0.t == 0
        assert out.obs.shape == (4, 84, 84, 3) and out.reward.shape == (4,)
        assert not out.done.any()
        s1b, out_b = E.step(env, s0, act)  # pure: same inputs, same outputs
        assert torch.equal(out.obs, out_b.obs) and torch.equal(s1.sys.qpos, s1b.sys.qpos)
        assert torch.equal(E.observe(env, s1), out.obs)
        with pytest.raises(ValueError):
            E.step(env, s0, np.zeros((3, env.n_joints)))

    def test_step_obs_is_render_of_state(self, E, oracle):
        """step()'s observation equals the oracle's render of the env's own
        (device) poses with the advanced distractor state."""
        env, s, _ = _env(E, "ant_lite", batch=8, seed=2, distractor_mode="color")
        rng = np.random.default_rng(0)
        for t in range(3):
            s, out = E.step(env, s, rng.uniform(-1, 1, (8, env.n_joints)))
        poses = env.poses(s.sys).cpu().numpy()
        px, _ = oracle.render_robot_batch(env.geometry, poses, 84, 84, False, threads=4)
        oracle.apply_color_inplace(px, s.distractor.color_bias.cpu().numpy())
        np.testing.assert_array_equal(out.obs.cpu().numpy(), px)

    def test_walker_falls_resets_and_bookkeeping(self, E, tmp_path):
        import torch

        from paper_2502_00021_b200.bench_support import synthetic_pack
        from paper_2502_00021_b200.video_pack import save_video_pack

        path = tmp_path / "p.pxvp"
        save_video_pack(synthetic_pack(), path)
        env, s, _ = _env(E, "walker_lite", batch=16, seed=1, distractor_mode="video",
                         video_pack_path=str(path))
        rng = np.random.default_rng(1)
        saw_done = False
        total = torch.zeros(16, dtype=torch.float64, device="cuda")
        for t in range(150):
            prev_vid = s.distractor.video_index.clone()
            s, out = E.step(env, s, rng.uniform(-1, 1, (16, env.n_joints)))
            total += out.reward
            d = out.done
            if d.any():
                saw_done = True
                assert (s.distractor.frame_cursor[d] == 0).all()
                assert (s.sys.step_count[d] == 0).all()
                assert (out.info["episode_length"][d] > 0).all()
                assert (s.episode_length[d] == 0).all()
            assert (out.info["episode_length"][~d] == 0).all()
            _ = prev_vid
        assert saw_done, "walker should fall under random actions within 150 steps"

    def test_slice_impersonation(self, E):
        import torch

        big_env, big, _ = _env(E, "hopper_lite", batch=12, seed=4, distractor_mode="color")
        part_env, part, _ = _env(E, "hopper_lite", batch=4, seed=4, distractor_mode="color",
                                 env_offset=8, logical_batch=12)
        rng = np.random.default_rng(2)
        for t in range(20):
            a = rng.uniform(-1, 1, (12, big_env.n_joints))
            big, ob = E.step(big_env, big, a)
            part, op = E.step(part_env, part, a[8:12])
            assert torch.equal(ob.obs[8:12], op.obs)
            assert torch.equal(big.sys.qpos[8:12], part.sys.qpos)

    def test_grayscale_formula(self, E):
        import torch

        _, _, rgb = _env(E, "cheetah_lite", batch=2, seed=5)
        _, _, gray = _env(E, "cheetah_lite", batch=2, seed=5, observation="grayscale")
        p = rgb.to(torch.int64)
        want = ((299 * p[..., 0] + 587 * p[..., 1] + 114 * p[..., 2] + 500) // 1000)
        assert torch.equal(gray[..., 0].to(torch.int64), want)

    def test_render_frame_background_mask(self, E, tmp_path):
        """Video foreground equals mode none (reference tests/test_env.py:226-239)."""
        import torch

        from paper_2502_00021_b200.bench_support import synthetic_pack
        from paper_2502_00021_b200.video_pack import save_video_pack

        path = tmp_path / "p.pxvp"
        save_video_pack(synthetic_pack(), path)
        env_v, sv, ov = _env(E, "walker_lite", batch=3, seed=6, distractor_mode="video",
                             video_pack_path=str(path))
        env_n, sn, on = _env(E, "walker_lite", batch=3, seed=6, floor_in_background=True)
        fr = env_v._render_frame(sv.sys, sv.distractor)
        fg = ~fr.background_mask
        assert fg.any()
        assert torch.equal(ov[fg], on[fg])


@pytest.mark.parametrize("name,mode,batch", [("walker_lite", "video", 24), ("cheetah_lite", "none", 3),
                                              ("hopper_lite", "color", 200)])
def test_step_loop_same_without_programmatic_launch(E, knobs, name, mode, batch, tmp_path):
    """The render launch with programmatic dependent launch (the default:
    it may be scheduled while the physics / FK kernels before it run, and
    waits for them before reading) against plain launches: the same obs,
    rewards and state over a stretch of steps with resets."""
    import torch

    from paper_2502_00021_b200.bench_support import synthetic_pack
    from paper_2502_00021_b200.video_pack import save_video_pack

    kw = {}
    if mode == "video":
        path = tmp_path / "p.pxvp"
        save_video_pack(synthetic_pack(), path)
        kw["video_pack_path"] = str(path)
    runs = []
    for no_pdl in (None, 1):
        knobs.set("PXR_DEBUG_NO_PDL", no_pdl)
        env, s, obs = _env(E, name, batch=batch, seed=5, distractor_mode=mode, **kw)
        gen = torch.Generator(device="cuda").manual_seed(1)
        frames = [obs.clone()]
        for _ in range(40):
            act = torch.rand((batch, env.n_joints), generator=gen, device="cuda",
                             dtype=torch.float64) * 2 - 1
            s, out = E.step(env, s, act)
            frames.append(out.obs.clone())
        torch.cuda.synchronize()
        runs.append((frames, s.sys.qpos.clone(), s.sys.qvel.clone()))
    (fa, qa, va), (fb, qb, vb) = runs
    for a, b in zip(fa, fb):
        assert torch.equal(a, b)
    assert torch.equal(qa, qb) and torch.equal(va, vb)


class TestStepGraph:
    """StepGraph (policy -> step captured as one CUDA graph, replayed with the
    step key computed on the device) against the pure ``step`` loop."""

    @pytest.mark.parametrize("name,mode,extra", [
        ("walker_lite", "video", {}), ("hopper_lite", "color", {}), ("cheetah_lite", "none", {}),
        ("walker_lite", "video", {"observation": "grayscale", "logical_batch": 96,
                                  "env_offset": 48}),
    ])
    def test_replay_equals_step_loop(self, E, name, mode, extra, tmp_path):
        import torch

        from paper_2502_00021_b200.bench import ConvStub, conv_stub_forward
        from paper_2502_00021_b200.bench_support import synthetic_pack
        from paper_2502_00021_b200.video_pack import save_video_pack

        kw = dict(extra)
        if mode == "video":
            path = tmp_path / "p.pxvp"
            save_video_pack(synthetic_pack(), path)
            kw["video_pack_path"] = str(path)
        # long enough for walker falls: resets + video re-draws (PXR_SOAK_STEPS
        # lengthens it for soak runs)
        B, T = 24, int(os.environ.get("PXR_SOAK_STEPS", "120"))
        env, s0, obs0 = _env(E, name, batch=B, seed=3, distractor_mode=mode, **kw)
        stub = ConvStub.create(84, 84, int(obs0.shape[-1]), env.n_joints, seed=0)
        # reference: the pure step loop
        s, obs = s0, obs0
        saw_done = False
        for _ in range(T):
            s, out = E.step(env, s, conv_stub_forward(stub, obs))
            obs = out.obs
            saw_done |= bool(out.done.any())
        # graph replay on an independent copy of the initial state
        g_state = dataclasses.replace(
            s0, sys=s0.sys.copy(), distractor=s0.distractor.copy(),
            episode_return=s0.episode_return.clone(), episode_length=s0.episode_length.clone())
        g = E.StepGraph(env, g_state, obs0.clone(), lambda o: conv_stub_forward(stub, o))
        g.replay(T - 1)
        g.replay(1)
        torch.cuda.synchronize()
        assert g_state.t == s.t == T
        assert torch.equal(g.obs, obs)
        assert torch.equal(g_state.sys.qpos, s.sys.qpos)
        assert torch.equal(g_state.sys.qvel, s.sys.qvel)
        assert torch.equal(g_state.sys.step_count, s.sys.step_count)
        assert torch.equal(g_state.episode_return, s.episode_return)
        assert torch.equal(g_state.episode_length, s.episode_length)
        assert torch.equal(g.reward, out.reward)
        assert torch.equal(g.done.bool(), out.done)
        assert torch.equal(g.info_length, out.info["episode_length"])
        for f in ("color_bias", "video_index", "frame_cursor", "direction", "frame_count"):
            a, b = getattr(g_state.distractor, f, None), getattr(s.distractor, f, None)
            if a is not None:
                assert torch.equal(a, b), f
        if name == "walker_lite":
            assert saw_done, "the loop should include resets"

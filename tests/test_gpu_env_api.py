"""The reference's Env behaviour tests (tests/test_env.py:29-247) restated
against this package's device-resident Env: make_env purity / shapes / seeds
/ errors, step advance + reward + purity, observe == step obs, action repeat,
shape errors, action clamping, the in-band auto-reset convention and its
episode bookkeeping, and the distractor modes."""

import dataclasses

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def E():
    import importlib

    return importlib.import_module("paper_2502_00021_b200.env")


@pytest.fixture(scope="module")
def pack_path(tmp_path_factory):
    from paper_2502_00021_b200.bench_support import synthetic_pack
    from paper_2502_00021_b200.video_pack import save_video_pack

    p = tmp_path_factory.mktemp("pack") / "pack.pxvp"
    save_video_pack(synthetic_pack(), p)
    return str(p)


def random_actions(env, t, seed=123):
    """Per-env action stream that depends only on the env's global index."""
    from paper_2502_00021_b200.prng import fold_in, key_from_seed, uniform

    k = fold_in(key_from_seed(seed), t)
    cfg = env.config
    return np.stack([uniform(fold_in(k, cfg.env_offset + i), env.n_joints, -1.0, 1.0)
                     for i in range(cfg.batch)])


def host(x):
    return x.cpu().numpy()


class TestMake:
    def test_purity_shapes_seeds(self, E):
        cfg = E.EnvConfig(model="hopper_lite", batch=2, seed=3)
        _, s1, o1 = E.make_env(cfg)
        _, s2, o2 = E.make_env(cfg)
        assert np.array_equal(host(o1), host(o2))
        assert np.array_equal(host(s1.sys.qpos), host(s2.sys.qpos))
        env, _, obs = E.make_env(E.EnvConfig(batch=3, width=32, height=24))
        assert tuple(obs.shape) == (3, 24, 32, 3) and env.obs_shape == (24, 32, 3)
        _, _, g = E.make_env(E.EnvConfig(batch=2, width=32, height=32,
                                         observation="grayscale"))
        assert tuple(g.shape) == (2, 32, 32, 1)
        _, _, a = E.make_env(E.EnvConfig(batch=1, seed=0))
        _, _, b = E.make_env(E.EnvConfig(batch=1, seed=1))
        assert not np.array_equal(host(a), host(b))

    def test_errors(self, E):
        with pytest.raises(ValueError, match="builtin"):
            E.make_env(E.EnvConfig(model="no_such_model"))
        with pytest.raises(ValueError, match="video_pack_path"):
            E.make_env(E.EnvConfig(distractor_mode="video"))


class TestStep:
    def test_step_advances_rewards_and_purity(self, E):
        env, state, _ = E.make_env(E.EnvConfig(model="cheetah_lite", batch=2, seed=1))
        s, out = E.step(env, state, np.zeros((2, env.n_joints)))
        assert s.t == 1 and tuple(out.obs.shape) == (2, 84, 84, 3)
        assert tuple(out.reward.shape) == (2,) and not bool(out.done.any())
        cfg = E.EnvConfig(model="hopper_lite", batch=2, seed=2, width=32, height=32)
        env1, st1, _ = E.make_env(cfg)
        env2, st2, _ = E.make_env(cfg)
        acts = random_actions(env1, 0)
        _, a = E.step(env1, st1, acts)
        _, b = E.step(env2, st2, acts)
        assert np.array_equal(host(a.obs), host(b.obs))
        assert np.array_equal(host(a.reward), host(b.reward))

    def test_observe_matches_step_obs(self, E):
        env, state, _ = E.make_env(E.EnvConfig(batch=2, seed=4, width=32, height=32))
        for t in range(3):
            state, out = E.step(env, state, random_actions(env, t))
        assert np.array_equal(host(E.observe(env, state)), host(out.obs))

    def test_action_repeat_accumulates_reward(self, E):
        base = E.EnvConfig(model="cheetah_lite", batch=1, seed=6, width=32, height=32)
        env1, s1, _ = E.make_env(base)
        env2, s2, _ = E.make_env(dataclasses.replace(base, action_repeat=2))
        acts = np.full((1, env1.n_joints), 0.5)
        s1, o1 = E.step(env1, s1, acts)
        s1, o1b = E.step(env1, s1, acts)
        s2, o2 = E.step(env2, s2, acts)
        assert np.array_equal(host(s1.sys.qpos), host(s2.sys.qpos))
        assert float(o2.reward[0]) == pytest.approx(float(o1.reward[0] + o1b.reward[0]))

    def test_shape_mismatch_and_clamping(self, E):
        env, state, _ = E.make_env(E.EnvConfig(batch=2))
        with pytest.raises(ValueError):
            E.step(env, state, np.zeros((2, env.n_joints + 1)))
        env, state, _ = E.make_env(E.EnvConfig(batch=1, seed=7, width=32, height=32))
        _, a = E.step(env, state, np.full((1, env.n_joints), 9.0))
        _, b = E.step(env, state, np.ones((1, env.n_joints)))
        assert np.array_equal(host(a.obs), host(b.obs))
        assert np.array_equal(host(a.reward), host(b.reward))


class TestAutoReset:
    def test_episode_boundary(self, E):
        env, state, _ = E.make_env(E.EnvConfig(model="cheetah_lite", batch=1, seed=8,
                                               width=32, height=32))
        assert env.spec.episode_length == 1000
        state.sys.step_count.fill_(999)  # fast-forward instead of stepping 1000 times
        state, out = E.step(env, state, np.zeros((1, env.n_joints)))
        assert bool(out.done[0]) and int(out.info["episode_length"][0]) > 0
        # in-band convention: the obs already belongs to the new episode
        assert int(state.sys.step_count[0]) == 0 and int(state.episode_length[0]) == 0
        assert float(state.episode_return[0]) == 0.0

    def test_walker_fall_terminates(self, E):
        env, state, _ = E.make_env(E.EnvConfig(model="walker_lite", batch=1, seed=9,
                                               width=32, height=32))
        for t in range(300):
            state, out = E.step(env, state, random_actions(env, t))
            if bool(out.done[0]):
                assert int(out.info["episode_length"][0]) == t + 1
                break
        else:
            pytest.fail("random walker should fall within 300 steps")

    def test_info_zero_when_not_done_and_running_totals(self, E):
        env, state, _ = E.make_env(E.EnvConfig(batch=2, seed=10, width=32, height=32))
        state, out = E.step(env, state, np.zeros((2, env.n_joints)))
        assert not bool(out.done.any())
        assert bool((out.info["episode_return"] == 0.0).all())
        assert bool((out.info["episode_length"] == 0).all())
        env, state, _ = E.make_env(E.EnvConfig(batch=1, seed=11, width=32, height=32))
        total = 0.0
        for t in range(5):
            state, out = E.step(env, state, random_actions(env, t))
            total += float(out.reward[0])
        assert float(state.episode_return[0]) == pytest.approx(total)
        assert int(state.episode_length[0]) == 5


class TestDistractorModes:
    def test_color_mode_changes_pixels(self, E):
        base = E.EnvConfig(batch=1, seed=15, width=32, height=32)
        _, _, plain = E.make_env(base)
        _, _, colored = E.make_env(dataclasses.replace(base, distractor_mode="color"))
        assert not np.array_equal(host(plain), host(colored))

    def test_video_foreground_matches_none(self, E, pack_path):
        base = E.EnvConfig(batch=1, seed=16, width=32, height=32, floor_in_background=True)
        env_n, state_n, obs_n = E.make_env(base)
        _, _, obs_v = E.make_env(dataclasses.replace(base, distractor_mode="video",
                                                     video_pack_path=pack_path))
        fg = ~host(env_n._render_frame(state_n.sys, state_n.distractor).background_mask)
        on, ov = host(obs_n), host(obs_v)
        assert np.array_equal(on[fg], ov[fg]) and np.any(on[~fg] != ov[~fg])

    def test_video_floor_defaults_to_background(self, E, pack_path):
        cfg = E.EnvConfig(distractor_mode="video", video_pack_path=pack_path)
        assert cfg.resolved_floor_in_background is True
        assert E.EnvConfig().resolved_floor_in_background is False

"""Env behaviour the reference pins in tests/test_env.py:29-247, checked
against this package's device-resident Env: construction (deterministic,
shapes, seeds matter, errors), stepping (counter, reward shape, purity,
observe == last obs, action repeat sums rewards, bad action shapes, action
clamping), the in-band auto-reset with its episode bookkeeping, and how the
distractor modes change (or do not change) the observation."""

import dataclasses

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SMALL = dict(width=32, height=32)


@pytest.fixture(scope="module")
def E():
    import importlib

    return importlib.import_module("paper_2502_00021_b200.env")


@pytest.fixture(scope="module")
def pack_file(tmp_path_factory):
    from paper_2502_00021_b200.bench_support import synthetic_pack
    from paper_2502_00021_b200.video_pack import save_video_pack

    out = tmp_path_factory.mktemp("packs") / "synthetic.pxvp"
    save_video_pack(synthetic_pack(), out)
    return str(out)


def np_(t):
    return t.detach().cpu().numpy()


def actions_for(env, t, seed=123):
    """Actions that depend only on (seed, t, global env index)."""
    from paper_2502_00021_b200.prng import fold_in, key_from_seed, uniform

    base = fold_in(key_from_seed(seed), t)
    off = env.config.env_offset
    return np.stack([uniform(fold_in(base, off + i), env.n_joints, -1.0, 1.0)
                     for i in range(env.config.batch)])


def fresh(E, **kw):
    return E.make_env(E.EnvConfig(**kw))


def test_construction(E):
    (_, s1, o1), (_, s2, o2) = (fresh(E, model="hopper_lite", batch=2, seed=3) for _ in range(2))
    assert np.array_equal(np_(o1), np_(o2)) and np.array_equal(np_(s1.sys.qpos), np_(s2.sys.qpos))
    env, _, obs = fresh(E, batch=3, width=32, height=24)
    assert tuple(obs.shape) == (3, 24, 32, 3) and env.obs_shape == (24, 32, 3)
    assert tuple(fresh(E, batch=2, observation="grayscale", **SMALL)[2].shape) == (2, 32, 32, 1)
    assert not np.array_equal(np_(fresh(E, batch=1, seed=0)[2]), np_(fresh(E, batch=1, seed=1)[2]))
    for kw, msg in (({"model": "no_such_model"}, "builtin"),
                    ({"distractor_mode": "video"}, "video_pack_path")):
        with pytest.raises(ValueError, match=msg):
            fresh(E, **kw)


def test_stepping(E):
    env, state, _ = fresh(E, model="cheetah_lite", batch=2, seed=1)
    nxt, out = E.step(env, state, np.zeros((2, env.n_joints)))
    assert nxt.t == 1 and tuple(out.obs.shape) == (2, 84, 84, 3)
    assert tuple(out.reward.shape) == (2,) and not bool(out.done.any())
    # purity: two identical envs, same actions, same outputs
    cfg = dict(model="hopper_lite", batch=2, seed=2, **SMALL)
    (e1, st1, _), (e2, st2, _) = fresh(E, **cfg), fresh(E, **cfg)
    acts = actions_for(e1, 0)
    r1, r2 = E.step(e1, st1, acts)[1], E.step(e2, st2, acts)[1]
    assert np.array_equal(np_(r1.obs), np_(r2.obs)) and np.array_equal(np_(r1.reward),
                                                                         np_(r2.reward))
    # observe() re-renders the last step's observation
    env, state, _ = fresh(E, batch=2, seed=4, **SMALL)
    for t in range(3):
        state, out = E.step(env, state, actions_for(env, t))
    assert np.array_equal(np_(E.observe(env, state)), np_(out.obs))


def test_action_repeat_shapes_and_clamping(E):
    base = E.EnvConfig(model="cheetah_lite", batch=1, seed=6, **SMALL)
    e1, s1, _ = E.make_env(base)
    e2, s2, _ = E.make_env(dataclasses.replace(base, action_repeat=2))
    half = np.full((1, e1.n_joints), 0.5)
    s1, a = E.step(e1, s1, half)
    s1, b = E.step(e1, s1, half)
    s2, c = E.step(e2, s2, half)
    assert np.array_equal(np_(s1.sys.qpos), np_(s2.sys.qpos))
    assert float(c.reward[0]) == pytest.approx(float(a.reward[0] + b.reward[0]))
    env, state, _ = fresh(E, batch=2)
    with pytest.raises(ValueError):
        E.step(env, state, np.zeros((2, env.n_joints + 1)))
    env, state, _ = fresh(E, batch=1, seed=7, **SMALL)
    big, unit = (E.step(env, state, np.full((1, env.n_joints), v))[1] for v in (9.0, 1.0))
    assert np.array_equal(np_(big.obs), np_(unit.obs))
    assert np.array_equal(np_(big.reward), np_(unit.reward))


def test_auto_reset(E):
    env, state, _ = fresh(E, model="cheetah_lite", batch=1, seed=8, **SMALL)
    assert env.spec.episode_length == 1000
    state.sys.step_count.fill_(999)  # jump to the last step of the episode
    state, out = E.step(env, state, np.zeros((1, env.n_joints)))
    assert bool(out.done[0]) and int(out.info["episode_length"][0]) > 0
    # the returned state (and obs) already belong to the next episode
    assert (int(state.sys.step_count[0]), int(state.episode_length[0]),
            float(state.episode_return[0])) == (0, 0, 0.0)
    env, state, _ = fresh(E, model="walker_lite", batch=1, seed=9, **SMALL)
    fell_at = None
    for t in range(300):
        state, out = E.step(env, state, actions_for(env, t))
        if bool(out.done[0]):
            fell_at = t
            assert int(out.info["episode_length"][0]) == t + 1
            break
    assert fell_at is not None, "random walker should fall within 300 steps"
    env, state, _ = fresh(E, batch=2, seed=10, **SMALL)
    _, out = E.step(env, state, np.zeros((2, env.n_joints)))
    assert not bool(out.done.any())
    assert bool((out.info["episode_return"] == 0).all() and (out.info["episode_length"] == 0).all())
    env, state, _ = fresh(E, batch=1, seed=11, **SMALL)
    running = 0.0
    for t in range(5):
        state, out = E.step(env, state, actions_for(env, t))
        running += float(out.reward[0])
    assert float(state.episode_return[0]) == pytest.approx(running)
    assert int(state.episode_length[0]) == 5


def test_distractor_modes(E, pack_file):
    base = E.EnvConfig(batch=1, seed=15, **SMALL)
    assert not np.array_equal(np_(E.make_env(base)[2]),
                              np_(E.make_env(dataclasses.replace(base,
                                                                 distractor_mode="color"))[2]))
    plain_cfg = E.EnvConfig(batch=1, seed=16, floor_in_background=True, **SMALL)
    env_n, state_n, obs_n = E.make_env(plain_cfg)
    obs_v = E.make_env(dataclasses.replace(plain_cfg, distractor_mode="video",
                                           video_pack_path=pack_file))[2]
    fg = ~np_(env_n._render_frame(state_n.sys, state_n.distractor).background_mask)
    a, b = np_(obs_n), np_(obs_v)
    assert np.array_equal(a[fg], b[fg]) and (a[~fg] != b[~fg]).any()
    assert E.EnvConfig(distractor_mode="video",
                       video_pack_path=pack_file).resolved_floor_in_background is True
    assert E.EnvConfig().resolved_floor_in_background is False

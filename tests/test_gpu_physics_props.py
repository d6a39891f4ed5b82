"""The reference's physics property tests (tests/test_physics.py:100-340)
restated for this package's device physics: static equilibrium on the
contact springs, the reward terms, termination, reset draws (purity, noise
bounds, env_offset slices), batch semantics (purity, order equivariance,
batch-size independence, action clamping, shape errors, episode length) and
forward kinematics (root passthrough, translation equivariance, hand
oracles, shape errors)."""

import dataclasses

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

CONTACT_SPRING = 4000.0  # reference physics.py contact stiffness (csrc/pxr_physics.cu)


@pytest.fixture(scope="module")
def P():
    import importlib

    return importlib.import_module("paper_2502_00021_b200.physics")


@pytest.fixture(scope="module")
def M():
    import importlib

    return importlib.import_module("paper_2502_00021_b200.models")


def free_link(M, dt=1e-3, substeps=5):
    return M.ModelSpec("stick", (M.LinkSpec(length=1.0, mass=2.0, radius=0.05),), (), dt=dt,
                       substeps=substeps)


def state_from_qpos(P, torch, qpos, qvel=None):
    """A SystemState on the device from host generalized coordinates."""
    q = np.atleast_2d(np.asarray(qpos, dtype=np.float64))
    v = np.zeros_like(q) if qvel is None else np.atleast_2d(np.asarray(qvel, dtype=np.float64))
    b = q.shape[0]
    return P.SystemState(torch.from_numpy(q.copy()).cuda(), torch.from_numpy(v.copy()).cuda(),
                         torch.zeros(b, dtype=torch.int64, device="cuda"),
                         torch.zeros(b, dtype=torch.uint8, device="cuda"))


def host(x):
    return x.cpu().numpy()


def test_resting_link_is_stationary(P, M, torch):
    spec = free_link(M)
    pen = spec.links[0].mass * P.GRAVITY / (2.0 * CONTACT_SPRING)  # both end springs share it
    s = state_from_qpos(P, torch, [0.0, -pen, 0.0])
    acts = np.zeros((1, 0))
    for _ in range(2000):  # the damper kills any residual motion
        s = P.step_dynamics(spec, s, acts)
    before = host(s.qpos)
    s = P.step_dynamics(spec, s, acts)
    assert np.max(np.abs(host(s.qpos) - before)) < 1e-6


def test_reward_terms_and_termination(P, M, torch):
    ch = M.builtin_model("cheetah_lite")
    rest = state_from_qpos(P, torch, ch.rest()[None])
    reward = lambda spec, a, b, u: host(P.compute_reward(spec, a, b, u))  # noqa: E731
    # (spec, prev, next, actions) -> expected reward
    glide = dataclasses.replace(free_link(M), dt=0.05, forward_weight=1.0)
    table = [
        (ch, rest, rest, np.zeros((1, 6)), 0.0),
        (glide, state_from_qpos(P, torch, [0.0, 1.0, 0.0]),
         state_from_qpos(P, torch, [0.1, 1.0, 0.0]), np.zeros((1, 0)), 2.0),  # 0.1 / 0.05
        (ch, rest, rest, np.array([[1.0, -1.0] * 3]), -0.6),  # ctrl cost 0.1 x six joints
    ]
    for spec, a, b, u, want in table:
        assert float(reward(spec, a, b, u)[0]) == pytest.approx(want)
    assert np.array_equal(reward(ch, rest, rest, np.full((1, 6), 50.0)),
                          reward(ch, rest, rest, np.ones((1, 6))))  # actions clamp to [-1, 1]
    heights = np.tile(ch.rest(), (3, 1))
    heights[:, 1] = (-5.0, 0.0, 5.0)  # the cheetah never terminates
    assert not host(P.check_termination(ch, state_from_qpos(P, torch, heights))).any()
    wk = M.builtin_model("walker_lite")
    for z, terminated in ((0.5, True), (0.8, False)):  # below 0.8 only (strict)
        q = wk.rest()[None].copy()
        q[0, 1] = z
        assert bool(host(P.check_termination(wk, state_from_qpos(P, torch, q)))[0]) is terminated


def test_reset_draws(P, M, pkg):
    seed = pkg.key_from_seed
    walker, hopper, cheetah = (M.builtin_model(n) for n in ("walker_lite", "hopper_lite",
                                                             "cheetah_lite"))
    first, again = (P.reset_state(walker, seed(0), 4) for _ in range(2))
    for field in ("qpos", "qvel"):
        assert np.array_equal(host(getattr(first, field)), host(getattr(again, field)))
    pair = host(P.reset_state(walker, seed(1), 2).qpos)
    assert not np.array_equal(pair[0], pair[1])
    many = P.reset_state(hopper, seed(2), 64)
    assert np.abs(host(many.qpos) - hopper.rest()).max() <= 0.1  # U(-0.1, 0.1) around rest
    assert not host(many.done).any() and not host(many.step_count).any()
    whole, last3 = P.reset_state(cheetah, seed(3), 10), P.reset_state(cheetah, seed(3), 3,
                                                                      env_offset=7)
    for field in ("qpos", "qvel"):  # env_offset reproduces the batch slice
        assert np.array_equal(host(getattr(whole, field))[7:], host(getattr(last3, field)))
    with pytest.raises(ValueError):
        P.reset_state(cheetah, seed(3), 0)


def _policy_actions(pkg, spec, seed, t, env_ids):
    from paper_2502_00021_b200.prng import fold_in, uniform

    step_key = fold_in(pkg.key_from_seed(seed), t)
    return np.stack([uniform(fold_in(step_key, e), spec.n_joints, -1.0, 1.0) for e in env_ids])


def test_batch_semantics(P, M, pkg, torch):
    hop = M.builtin_model("hopper_lite")
    s0 = P.reset_state(hop, pkg.key_from_seed(4), 3)
    u = np.full((3, hop.n_joints), 0.3)
    assert np.array_equal(host(P.step_dynamics(hop, s0, u).qpos),
                          host(P.step_dynamics(hop, s0, u).qpos))  # pure
    wk = M.builtin_model("walker_lite")
    s8 = P.reset_state(wk, pkg.key_from_seed(5), 8)
    g = np.random.default_rng(0)
    u8 = g.uniform(-1, 1, (8, wk.n_joints))
    order = g.permutation(8)
    idx = torch.from_numpy(order).cuda()
    shuffled = P.SystemState(*(getattr(s8, f)[idx] for f in ("qpos", "qvel", "step_count",
                                                            "done")))
    ref, perm = P.step_dynamics(wk, s8, u8), P.step_dynamics(wk, shuffled, u8[order])
    for field in ("qpos", "qvel"):  # permuting the batch permutes the results
        assert np.array_equal(host(getattr(perm, field)), host(getattr(ref, field))[order])
    ch = M.builtin_model("cheetah_lite")
    batch16 = P.reset_state(ch, pkg.key_from_seed(6), 16)
    k = 11
    solo = P.SystemState(*(getattr(batch16, f)[k:k + 1].clone()
                           for f in ("qpos", "qvel", "step_count", "done")))
    for t in range(50):  # env k alone steps exactly like env k of 16
        batch16 = P.step_dynamics(ch, batch16, _policy_actions(pkg, ch, 7, t, range(16)))
        solo = P.step_dynamics(ch, solo, _policy_actions(pkg, ch, 7, t, [k]))
    for field in ("qpos", "qvel"):
        assert np.array_equal(host(getattr(solo, field))[0], host(getattr(batch16, field))[k])


def test_action_limits_shapes_and_episode_length(P, M, pkg, torch):
    hop = M.builtin_model("hopper_lite")
    s0 = P.reset_state(hop, pkg.key_from_seed(10), 2)
    ten, one = (P.step_dynamics(hop, s0, np.full((2, hop.n_joints), v)) for v in (10.0, 1.0))
    assert np.array_equal(host(ten.qpos), host(one.qpos))
    with pytest.raises(ValueError):
        P.step_dynamics(hop, s0, np.zeros((2, hop.n_joints + 1)))
    short = dataclasses.replace(free_link(M), episode_length=3)
    s = state_from_qpos(P, torch, [0.0, 5.0, 0.0])
    flags = []
    for _ in range(3):
        flags.append(bool(s.done[0]))
        s = P.step_dynamics(short, s, np.zeros((1, 0)))
    assert flags == [False] * 3 and bool(s.done[0]) and int(s.step_count[0]) == 3


def test_forward_kinematics(P, M):
    fk = lambda spec, q: P.forward_kinematics(spec, np.asarray(q, float)).cpu().numpy()  # noqa
    ch = M.builtin_model("cheetah_lite")
    assert np.array_equal(fk(ch, ch.rest()[None])[0, 0], ch.rest()[:3])  # root passes through
    wk = M.builtin_model("walker_lite")
    q = wk.rest()[None].copy()
    moved = q.copy()
    moved[0, :2] += (3.0, -0.5)
    a, b = fk(wk, q), fk(wk, moved)
    assert np.allclose(b[0, :, :2], a[0, :, :2] + (3.0, -0.5))
    assert np.array_equal(b[0, :, 2], a[0, :, 2])
    two_links = (M.LinkSpec(2.0, 1.0, 0.05), M.LinkSpec(1.0, 1.0, 0.05))
    # (anchor along the parent, qpos, expected child pose) worked by hand
    for anchor, qpos, child in ((1.0, (0.0, 0.0, 0.0, np.pi / 2), (2.0, 0.0, np.pi / 2)),
                                (0.5, (0.0, 0.0, np.pi / 2, 0.0), (0.0, 1.0, np.pi / 2))):
        spec = M.ModelSpec("hand", two_links, (M.JointSpec(0, -3.0, 3.0, 1.0, anchor=anchor),))
        assert np.allclose(fk(spec, [qpos])[0, 1], child)
    hop = M.builtin_model("hopper_lite")
    with pytest.raises(ValueError):
        fk(hop, np.zeros((1, hop.dof + 2)))

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


class TestRewardAndTermination:
    def test_reward_terms(self, P, M, torch):
        spec = M.builtin_model("cheetah_lite")
        s = state_from_qpos(P, torch, np.tile(spec.rest(), (1, 1)))
        assert float(P.compute_reward(spec, s, s, np.zeros((1, spec.n_joints)))[0]) == 0.0
        fl = dataclasses.replace(free_link(M), dt=0.05, forward_weight=1.0)
        a = state_from_qpos(P, torch, [0.0, 1.0, 0.0])
        b = state_from_qpos(P, torch, [0.1, 1.0, 0.0])
        assert float(P.compute_reward(fl, a, b, np.zeros((1, 0)))[0]) == pytest.approx(2.0)
        acts = np.array([[1.0, -1.0, 1.0, -1.0, 1.0, -1.0]])  # ctrl_cost 0.1, six joints
        assert float(P.compute_reward(spec, s, s, acts)[0]) == pytest.approx(-0.6)
        assert np.array_equal(host(P.compute_reward(spec, s, s, np.full((1, 6), 50.0))),
                              host(P.compute_reward(spec, s, s, np.ones((1, 6)))))

    def test_termination(self, P, M, torch):
        c = M.builtin_model("cheetah_lite")
        q = np.tile(c.rest(), (3, 1))
        q[:, 1] = [-5.0, 0.0, 5.0]
        assert not host(P.check_termination(c, state_from_qpos(P, torch, q))).any()
        w = M.builtin_model("walker_lite")
        q = np.tile(w.rest(), (1, 1))
        q[0, 1] = 0.5
        assert host(P.check_termination(w, state_from_qpos(P, torch, q)))[0]
        q[0, 1] = 0.8  # the boundary is strict
        assert not host(P.check_termination(w, state_from_qpos(P, torch, q)))[0]


class TestReset:
    def test_purity_difference_bounds(self, P, M, pkg):
        w = M.builtin_model("walker_lite")
        a, b = P.reset_state(w, pkg.key_from_seed(0), 4), P.reset_state(w, pkg.key_from_seed(0), 4)
        assert np.array_equal(host(a.qpos), host(b.qpos))
        assert np.array_equal(host(a.qvel), host(b.qvel))
        s = P.reset_state(w, pkg.key_from_seed(1), 2)
        assert not np.array_equal(host(s.qpos)[0], host(s.qpos)[1])
        h = M.builtin_model("hopper_lite")
        s = P.reset_state(h, pkg.key_from_seed(2), 64)
        assert np.max(np.abs(host(s.qpos) - h.rest())) <= 0.1
        assert not host(s.done).any() and np.all(host(s.step_count) == 0)

    def test_offset_slice_and_zero_batch(self, P, M, pkg):
        c = M.builtin_model("cheetah_lite")
        k = pkg.key_from_seed(3)
        big, tail = P.reset_state(c, k, 10), P.reset_state(c, k, 3, env_offset=7)
        assert np.array_equal(host(big.qpos)[7:], host(tail.qpos))
        assert np.array_equal(host(big.qvel)[7:], host(tail.qvel))
        with pytest.raises(ValueError):
            P.reset_state(c, k, 0)


class TestBatchSemantics:
    @staticmethod
    def _acts(pkg, spec, seed, t, ids):
        from paper_2502_00021_b200.prng import fold_in, uniform

        k = pkg.key_from_seed(seed)
        return np.stack([uniform(fold_in(fold_in(k, t), i), spec.n_joints, -1.0, 1.0)
                         for i in ids])

    def test_purity_and_order_equivariance(self, P, M, pkg, torch):
        h = M.builtin_model("hopper_lite")
        s0 = P.reset_state(h, pkg.key_from_seed(4), 3)
        acts = np.full((3, h.n_joints), 0.3)
        a, b = P.step_dynamics(h, s0, acts), P.step_dynamics(h, s0, acts)
        assert np.array_equal(host(a.qpos), host(b.qpos))
        w = M.builtin_model("walker_lite")
        s0 = P.reset_state(w, pkg.key_from_seed(5), 8)
        rng = np.random.default_rng(0)
        acts = rng.uniform(-1, 1, (8, w.n_joints))
        perm = rng.permutation(8)
        out = P.step_dynamics(w, s0, acts)
        pi = torch.from_numpy(perm).cuda()
        sp = P.SystemState(s0.qpos[pi], s0.qvel[pi], s0.step_count[pi], s0.done[pi])
        outp = P.step_dynamics(w, sp, acts[perm])
        assert np.array_equal(host(outp.qpos), host(out.qpos)[perm])
        assert np.array_equal(host(outp.qvel), host(out.qvel)[perm])

    def test_batch_size_independence(self, P, M, pkg):
        c = M.builtin_model("cheetah_lite")
        big = P.reset_state(c, pkg.key_from_seed(6), 16)
        i = 11
        one = P.SystemState(big.qpos[i:i + 1].clone(), big.qvel[i:i + 1].clone(),
                            big.step_count[i:i + 1].clone(), big.done[i:i + 1].clone())
        for t in range(50):
            big = P.step_dynamics(c, big, self._acts(pkg, c, 7, t, range(16)))
            one = P.step_dynamics(c, one, self._acts(pkg, c, 7, t, [i]))
        assert np.array_equal(host(one.qpos)[0], host(big.qpos)[i])
        assert np.array_equal(host(one.qvel)[0], host(big.qvel)[i])

    def test_clamp_shape_and_episode_length(self, P, M, pkg, torch):
        h = M.builtin_model("hopper_lite")
        s0 = P.reset_state(h, pkg.key_from_seed(10), 2)
        a = P.step_dynamics(h, s0, np.full((2, h.n_joints), 10.0))
        b = P.step_dynamics(h, s0, np.ones((2, h.n_joints)))
        assert np.array_equal(host(a.qpos), host(b.qpos))
        with pytest.raises(ValueError):
            P.step_dynamics(h, s0, np.zeros((2, h.n_joints + 1)))
        spec = dataclasses.replace(free_link(M), episode_length=3)
        s = state_from_qpos(P, torch, [0.0, 5.0, 0.0])
        for _ in range(3):
            assert not bool(s.done[0])
            s = P.step_dynamics(spec, s, np.zeros((1, 0)))
        assert bool(s.done[0]) and int(s.step_count[0]) == 3


class TestForwardKinematics:
    def test_root_and_translation(self, P, M):
        c = M.builtin_model("cheetah_lite")
        q = np.tile(c.rest(), (1, 1))
        assert np.array_equal(np.asarray(P.forward_kinematics(c, q).cpu())[0, 0], q[0, :3])
        w = M.builtin_model("walker_lite")
        q = np.tile(w.rest(), (1, 1))
        base = P.forward_kinematics(w, q).cpu().numpy()
        q2 = q.copy()
        q2[0, 0] += 3.0
        q2[0, 1] -= 0.5
        moved = P.forward_kinematics(w, q2).cpu().numpy()
        assert np.allclose(moved[0, :, 0], base[0, :, 0] + 3.0)
        assert np.allclose(moved[0, :, 1], base[0, :, 1] - 0.5)
        assert np.array_equal(moved[0, :, 2], base[0, :, 2])

    def test_hand_oracles_and_shape(self, P, M):
        elbow = M.ModelSpec("elbow", (M.LinkSpec(2.0, 1.0, 0.05), M.LinkSpec(1.0, 1.0, 0.05)),
                            (M.JointSpec(0, -3.0, 3.0, 1.0, anchor=1.0),))
        p = P.forward_kinematics(elbow, np.array([[0.0, 0.0, 0.0, np.pi / 2]])).cpu().numpy()
        assert np.allclose(p[0, 1], [2.0, 0.0, np.pi / 2])
        mid = M.ModelSpec("mid", (M.LinkSpec(2.0, 1.0, 0.05), M.LinkSpec(1.0, 1.0, 0.05)),
                          (M.JointSpec(0, -3.0, 3.0, 1.0, anchor=0.5),))
        p = P.forward_kinematics(mid, np.array([[0.0, 0.0, np.pi / 2, 0.0]])).cpu().numpy()
        assert np.allclose(p[0, 1], [0.0, 1.0, np.pi / 2])
        h = M.builtin_model("hopper_lite")
        with pytest.raises(ValueError):
            P.forward_kinematics(h, np.zeros((1, h.dof + 2)))

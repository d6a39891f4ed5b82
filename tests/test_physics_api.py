"""The reference's physics API on the device (reference physics.py; tests
modelled on tests/test_physics.py and the physics oracles of
tests/test_acceptance.py:206-245) and the video-pack tooling (reference
video_tools.py; tests/test_video_tools.py).

Physics numbers compare with tolerances (CUDA f64 cos/sin vs numpy; reset
draws are bit-exact); golden values come from the live reference
(tests/golden/physics.npz)."""

import numpy as np
import pytest

from conftest import MODEL_NAMES, golden, spec_of


def test_video_tools_roundtrip(tmp_path):
    import paper_2502_00021_b200 as P
    from paper_2502_00021_b200.video_tools import read_ppm, write_ppm

    rng = np.random.default_rng(0)
    root = tmp_path / "frames"
    for v, n in (("b", 3), ("a", 2)):
        (root / v).mkdir(parents=True)
        for i in range(n):
            write_ppm(rng.integers(0, 256, (10, 12, 3), dtype=np.uint8), root / v / f"{i:03d}.ppm")
    img = read_ppm(root / "a" / "000.ppm")
    assert img.shape == (10, 12, 3)
    (root / "a" / "bad.ppm").write_bytes(b"P5\n2 2\n255\n" + bytes(4))
    with pytest.raises(ValueError):
        read_ppm(root / "a" / "bad.ppm")
    (root / "a" / "bad.ppm").unlink()
    summary = P.pack_from_frames(str(root), str(tmp_path / "p.pxvp"), 8, 8)
    assert (summary.videos, summary.total_frames) == (2, 5)
    pack = P.load_video_pack(str(tmp_path / "p.pxvp"))
    assert list(pack.frame_counts) == [2, 3]  # subdirectories in name order
    rows, cols = P.nearest_map(8, 10), P.nearest_map(8, 12)
    np.testing.assert_array_equal(pack.flat_frames()[0][0], img[rows][:, cols])
    s = P.generate_synthetic_pack(P.key_from_seed(1), 2, 3, 8, 8, str(tmp_path / "s.pxvp"))
    assert (s.videos, s.total_frames) == (2, 6) and s.bytes > 0


@pytest.mark.gpu
class TestPhysicsAPI:
    @pytest.mark.parametrize("name", MODEL_NAMES)
    def test_step_reward_termination_vs_reference(self, pkg, torch, name):
        rec = golden("physics.npz")
        spec = spec_of(name)
        st = pkg.SystemState(torch.from_numpy(rec[f"{name}_qpos"]).cuda(),
                             torch.from_numpy(rec[f"{name}_qvel"]).cuda(),
                             torch.from_numpy(rec[f"{name}_steps"]).cuda(),
                             torch.zeros(32, dtype=torch.uint8, device="cuda"))
        act = rec[f"{name}_act"]
        nxt = pkg.step_dynamics(spec, st, act)
        assert nxt is not st and torch.equal(st.qpos, torch.from_numpy(rec[f"{name}_qpos"]).cuda())
        np.testing.assert_array_equal(nxt.qpos.cpu().numpy(), rec[f"{name}_qpos1"])
        np.testing.assert_array_equal(nxt.qvel.cpu().numpy(), rec[f"{name}_qvel1"])
        np.testing.assert_array_equal(nxt.done.cpu().numpy().astype(bool), rec[f"{name}_done1"])
        r = pkg.compute_reward(spec, st, nxt, act)
        np.testing.assert_array_equal(r.cpu().numpy(), rec[f"{name}_reward"])
        term = pkg.check_termination(spec, nxt).cpu().numpy()
        if spec.min_root_height is None:
            assert not term.any()
        else:
            np.testing.assert_array_equal(term, nxt.qpos[:, 1].cpu().numpy() < spec.min_root_height)
        with pytest.raises(ValueError):
            pkg.step_dynamics(spec, st, act[:, :-1] if act.shape[1] else np.zeros((32, 1)))

    @pytest.mark.parametrize("name", MODEL_NAMES)
    def test_warp_and_thread_kernels_agree_bitwise(self, pkg, torch, knobs, name):
        """pxr_physics_step has warp-per-env and half-warp-per-env kernels
        (small / medium batches) and a thread-per-env kernel (large); the same
        env must step
        identically in both (batch-size independence), contacts, limits and
        resets included: 60 control steps of random actions from the golden
        states."""
        rec = golden("physics.npz")
        spec = spec_of(name)
        rng = np.random.default_rng(11)
        acts = rng.uniform(-1.5, 1.5, (60,) + rec[f"{name}_act"].shape)
        finals = []
        for kind in ("warp", "thread", "half", "quarter"):
            knobs.set("PXR_DEBUG_PHYS", kind)
            st = pkg.SystemState(torch.from_numpy(rec[f"{name}_qpos"]).cuda(),
                                 torch.from_numpy(rec[f"{name}_qvel"]).cuda(),
                                 torch.from_numpy(rec[f"{name}_steps"]).cuda(),
                                 torch.zeros(32, dtype=torch.uint8, device="cuda"))
            rewards = []
            for a in acts:
                nxt = pkg.step_dynamics(spec, st, a)
                rewards.append(pkg.compute_reward(spec, st, nxt, a))
                st = nxt
            finals.append((st, torch.stack(rewards)))
        (a, ra) = finals[0]
        for b, rb in finals[1:]:  # (half falls back to warp for models with >= 16 dofs)
            assert torch.equal(a.qpos, b.qpos) and torch.equal(a.qvel, b.qvel)
            assert torch.equal(a.done, b.done) and torch.equal(a.step_count, b.step_count)
            assert torch.equal(ra, rb)

    @pytest.mark.parametrize("name", MODEL_NAMES)
    def test_reset_state_bit_exact(self, pkg, name):
        rec = golden("physics.npz")
        key = pkg.fold_in(pkg.key_from_seed(3), 0x5EED)
        st = pkg.reset_state(spec_of(name), key, 16, env_offset=5)
        np.testing.assert_array_equal(st.qpos.cpu().numpy(), rec[f"{name}_reset_qpos"])
        np.testing.assert_array_equal(st.qvel.cpu().numpy(), rec[f"{name}_reset_qvel"])
        with pytest.raises(ValueError):
            pkg.reset_state(spec_of(name), key, 0)

    def test_forward_kinematics_matches_host(self, pkg):
        from paper_2502_00021_b200.models import forward_kinematics_host

        spec = spec_of("humanoid_lite")
        q = np.random.default_rng(1).uniform(-1, 1, (9, spec.dof))
        got = pkg.forward_kinematics(spec, q).cpu().numpy()
        np.testing.assert_array_equal(got, forward_kinematics_host(spec, q))

    def test_ballistic_within_1e_3(self, pkg, torch):
        from paper_2502_00021_b200.models import LinkSpec, ModelSpec

        spec = ModelSpec("stick", (LinkSpec(1.0, 2.0, 0.05),), (), dt=1e-3, substeps=5)
        st = pkg.SystemState(torch.tensor([[0.0, 1.0, 0.0]], dtype=torch.float64, device="cuda"),
                             torch.zeros((1, 3), dtype=torch.float64, device="cuda"),
                             torch.zeros(1, dtype=torch.int64, device="cuda"),
                             torch.zeros(1, dtype=torch.uint8, device="cuda"))
        for _ in range(400):
            st = pkg.step_dynamics(spec, st, np.zeros((1, 0)))
        assert abs(float(st.qpos[0, 1]) - (1.0 - 0.5 * 9.81 * 0.4 ** 2)) <= 1e-3

    def test_pendulum_energy_drift_below_1_percent(self, pkg, torch):
        from paper_2502_00021_b200.models import JointSpec, LinkSpec, ModelSpec

        spec = ModelSpec("pendulum", (LinkSpec(1.0, 1.0, 0.05), LinkSpec(1.0, 5.0, 0.05)),
                         (JointSpec(0, -3.0, 3.0, 10.0),), dt=1e-3, substeps=1, fixed_root=True,
                         rest_qpos=(0.0, 2.0, 0.0, -1.2))
        st = pkg.SystemState(torch.from_numpy(spec.rest()[None, :].copy()).cuda(),
                             torch.zeros((1, 4), dtype=torch.float64, device="cuda"),
                             torch.zeros(1, dtype=torch.int64, device="cuda"),
                             torch.zeros(1, dtype=torch.uint8, device="cuda"))
        e0 = float(pkg.mechanical_energy(spec, st)[0])
        for _ in range(1000):
            st = pkg.step_dynamics(spec, st, np.zeros((1, 1)))
            e = float(pkg.mechanical_energy(spec, st)[0])
            assert abs(e - e0) < 0.01 * abs(e0)

"""The reference's renderer behaviour tests (tests/test_render.py:123-282)
restated against this package's device API: empty scene is sky, the floor
covers the lower half with the two checker colours, a triangle is visible
and masked, the nearer triangle wins whatever the draw order, pose
translation, render_batch equals single renders, the minimum resolution and
the 7 B/pixel memory budget, batch rows equal per-env renders, a robot is
visible."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def R():
    import importlib

    return importlib.import_module("paper_2502_00021_b200.render")


def front_camera(R):
    # looks down +y, so triangles in the y > 0 half-space are visible
    return R.Camera(eye=(0.0, -4.0, 1.0), target=(0.0, 0.0, 1.0))


def tri_mesh(R, p0, p1, p2, color):
    return R.Mesh(vertices=np.array([p0, p1, p2], dtype=np.float32),
                  triangles=np.array([[0, 1, 2]], dtype=np.int32), base_color=color)


def test_empty_scene_is_sky(R):
    f = R.render([], front_camera(R), floor_in_background=True, width=16, height=16)
    assert bool((f.pixels == f.pixels.new_tensor(R.SKY_COLOR)).all())
    assert bool(f.background_mask.all())


def test_floor_covers_lower_half(R):
    f = R.render([], front_camera(R), width=32, height=32)
    m = f.background_mask[0].cpu().numpy()
    assert m[:10].all() and not m[-10:].any()
    floor = f.pixels[0, -10:].reshape(-1, 3).cpu().numpy()
    assert {tuple(c) for c in np.unique(floor, axis=0)} == {R.FLOOR_DARK, R.FLOOR_LIGHT}


def test_triangle_visible_and_masked(R):
    mesh = tri_mesh(R, (-1, 0, 0.2), (1, 0, 0.2), (0, 0, 2.0), R.LINK_PALETTE[0])
    f = R.render([(mesh, R.Pose())], front_camera(R), floor_in_background=True, width=48,
                 height=48)
    covered = ~f.background_mask[0]
    assert 50 < int(covered.sum()) < 48 * 48 / 2
    assert bool(f.depth[0][covered].isfinite().all())


def test_nearer_triangle_wins_in_either_order(R):
    far_tri = tri_mesh(R, (-1, 1.0, 0.0), (1, 1.0, 0.0), (0, 1.0, 2.0), (1.0, 0.0, 0.0))
    near_tri = tri_mesh(R, (-1, -1.0, 0.0), (1, -1.0, 0.0), (0, -1.0, 2.0), (0.0, 1.0, 0.0))
    cam = front_camera(R)
    kw = dict(floor_in_background=True, width=32, height=32)
    a = R.render([(far_tri, R.Pose()), (near_tri, R.Pose())], cam, **kw)
    b = R.render([(near_tri, R.Pose()), (far_tri, R.Pose())], cam, **kw)
    assert bool((a.pixels == b.pixels).all())
    green = R.render([(near_tri, R.Pose())], cam, **kw).pixels[0, 16, 16]
    assert bool((a.pixels[0, 16, 16] == green).all())


def test_pose_translation(R):
    mesh = tri_mesh(R, (-0.5, 0, -0.5), (0.5, 0, -0.5), (0, 0, 0.5), R.LINK_PALETTE[1])
    cam = R.Camera(eye=(0.0, -4.0, 0.0), target=(0.0, 0.0, 0.0))
    kw = dict(floor_in_background=True, width=64, height=64)
    left = R.render([(mesh, R.Pose(x=-1.0))], cam, **kw)
    right = R.render([(mesh, R.Pose(x=1.0))], cam, **kw)
    cl = np.argwhere(~left.background_mask[0].cpu().numpy())
    cr = np.argwhere(~right.background_mask[0].cpu().numpy())
    assert cl[:, 1].mean() < 32 < cr[:, 1].mean()


def test_render_batch_matches_singles(R):
    meshes = [(tri_mesh(R, (-1, 0, 0), (1, 0, 0), (0, 0, 1.5), R.LINK_PALETTE[i]),
               R.Pose(x=0.3 * i)) for i in range(3)]
    scenes = [([m], front_camera(R)) for m in meshes]
    batch = R.render_batch(scenes, width=24, height=24)
    for i, (scene, cam) in enumerate(scenes):
        single = R.render(scene, cam, width=24, height=24)
        assert bool((batch.pixels[i] == single.pixels[0]).all())
        assert np.array_equal(batch.depth[i].cpu().numpy().view(np.uint32),
                              single.depth[0].cpu().numpy().view(np.uint32))


def test_minimum_resolution_and_memory_budget(R):
    with pytest.raises(ValueError):
        R.render([], front_camera(R), width=4, height=16)
    with pytest.raises(ValueError):
        R.Frame.allocate(1, 7, 64)
    f = R.Frame.allocate(5, 84, 84)
    total = f.pixels.numel() * f.pixels.element_size() + f.depth.numel() * f.depth.element_size()
    assert total == 5 * 84 * 84 * 7


def test_batch_matches_per_env_and_robot_visible(R):
    rng = np.random.default_rng(2)
    geom = R.RobotGeometry((0.5, 0.4), (0.05, 0.05))
    poses = np.zeros((4, 2, 3))
    poses[:, :, 0] = rng.uniform(-0.5, 0.5, (4, 2))
    poses[:, :, 1] = rng.uniform(0.3, 1.0, (4, 2))
    poses[:, :, 2] = rng.uniform(-np.pi, np.pi, (4, 2))
    cfg = R.CameraConfig()
    batch = R.render_robot_batch(geom, poses, cfg, 64, 64, False)
    for i in range(4):
        single = R.render_robot_batch(geom, poses[i:i + 1], cfg, 64, 64, False)
        assert bool((batch.pixels[i] == single.pixels[0]).all())
        assert np.array_equal(batch.depth[i].cpu().numpy().view(np.uint32),
                              single.depth[0].cpu().numpy().view(np.uint32))
    one = R.render_robot_batch(R.RobotGeometry((0.6,), (0.08,)), np.array([[[0.0, 0.6, 0.0]]]),
                               cfg, 84, 84, True)
    assert int((~one.background_mask[0]).sum()) > 20

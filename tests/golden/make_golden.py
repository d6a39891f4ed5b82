"""Generate the golden fixtures in tests/golden/ from the LIVE reference.

Run in the build container only (the reference tree is not on GPU boxes):

    PYTHONDONTWRITEBYTECODE=1 NUMBA_CACHE_DIR=/tmp/numba_cache \
    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Everything here calls the reference's own public functions
(pixelctrl.render.render_robot_batch, pixelctrl.distractor.*,
pixelctrl.env.make_env/step, pixelctrl.prng.*); the outputs are frozen
as .npz/.json fixtures that the CPU tests (oracle pinning) and the GPU
parity tests compare against.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))

import pixelctrl  # noqa: E402  (the reference, via PYTHONPATH)
from pixelctrl import distractor as D  # noqa: E402
from pixelctrl.env import EnvConfig, make_env, step  # noqa: E402
from pixelctrl.models import builtin_model, load_model  # noqa: E402
from pixelctrl.physics import forward_kinematics, model_arrays  # noqa: E402
from pixelctrl.prng import fold_in, key_from_seed  # noqa: E402
from pixelctrl.recorder import make_policy  # noqa: E402
from pixelctrl.render import (  # noqa: E402
    LINK_PALETTE, Camera, CameraConfig, Frame, Mesh, Pose, RobotGeometry, render, render_batch,
    render_robot_batch, tessellate_capsule, tessellate_sphere)
from pixelctrl.video_pack import VideoPack, save_video_pack  # noqa: E402
from pixelctrl.video_tools import generate_synthetic_pack  # noqa: E402

assert "/root/reference" in pixelctrl.__file__, pixelctrl.__file__

MODEL_DIR = os.path.join(REPO, "paper_2502_00021_b200", "assets", "models")
MODELS = {
    "cheetah_lite": "cheetah_lite",
    "walker_lite": "walker_lite",
    "hopper_lite": "hopper_lite",
    "ant_lite": os.path.join(MODEL_DIR, "ant_lite.model"),
    "humanoid_lite": os.path.join(MODEL_DIR, "humanoid_lite.model"),
}


def spec_of(name):
    m = MODELS[name]
    return builtin_model(m) if not m.endswith(".model") else load_model(m)


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def geometry_fixture():
    out = {}
    for name in MODELS:
        a = model_arrays(spec_of(name))
        g = RobotGeometry(a.length, a.radius)
        out[name] = {
            "n_verts": int(len(g.base_verts)), "n_tris": int(len(g.triangles)),
            "base_verts": sha(g.base_verts.astype(np.float32)),
            "vert_link": sha(g.vert_link.astype(np.int32)),
            "triangles": sha(g.triangles.astype(np.int32)),
            "tri_colors": sha(g.tri_colors.astype(np.float32)),
        }
    with open(os.path.join(HERE, "geometry.json"), "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)


def rollout_poses(name, batch, steps, seed, every):
    """Pose snapshots from the reference's own physics under random actions."""
    env, state, _ = make_env(EnvConfig(model=MODELS[name], batch=batch, seed=seed, threads=8))
    act = make_policy(f"random:{seed}", env)
    snaps = []
    for t in range(steps):
        state, _ = step(env, state, act(None, t))
        if t % every == every - 1:
            snaps.append(forward_kinematics(env.spec, state.sys.qpos))
    return np.stack(snaps)


def render_fixtures():
    rng = np.random.default_rng(7)
    for name in MODELS:
        spec = spec_of(name)
        a = model_arrays(spec)
        geom = RobotGeometry(a.length, a.radius)
        poses = rollout_poses(name, 16, 40, seed=3, every=20)  # (2, 16, L, 3)
        poses = poses.reshape(-1, spec.n_links, 3)
        wild = np.zeros((8, spec.n_links, 3))  # large angles (glibc |x| >= 120 path)
        wild[:, :, 0] = rng.uniform(-0.5, 0.5, (8, spec.n_links))
        wild[:, :, 1] = rng.uniform(0.3, 1.2, (8, spec.n_links))
        wild[:, :, 2] = rng.uniform(-300, 300, (8, spec.n_links))
        poses = np.concatenate([poses, wild])
        rec = {"poses": poses}
        for fib in (False, True):
            fr = render_robot_batch(geom, poses, CameraConfig(), 84, 84, fib, threads=8)
            rec[f"pixels_fib{int(fib)}"] = fr.pixels
            rec[f"depth_fib{int(fib)}"] = fr.depth
        fr = render_robot_batch(geom, poses[:8], CameraConfig(), 64, 48, False, threads=8)
        rec["pixels_64x48"] = fr.pixels
        rec["depth_64x48"] = fr.depth
        np.savez_compressed(os.path.join(HERE, f"render_{name}.npz"), **rec)


def small_pack(path, seed=11, videos=3, frames=5, size=16):
    generate_synthetic_pack(key_from_seed(seed), videos, frames, size, size, path)
    return pixelctrl.load_video_pack(path)


def distractor_fixtures():
    rec = {}
    k = key_from_seed(5)
    s = D.init_distractors("color", None, k, 64)
    rec["color_init_seed5_b64"] = s.color_bias
    s2 = D.init_distractors("color", None, k, 16, env_offset=48)
    rec["color_init_seed5_off48_b16"] = s2.color_bias
    kt = fold_in(key_from_seed(5), 3)
    rec["color_adv_seed5_t3_b64"] = D.advance_distractors(s, kt).color_bias
    rec["color_adv_seed5_t3_off48_b16"] = D.advance_distractors(s2, kt, env_offset=48).color_bias
    pack_path = os.path.join("/tmp", "golden_small.pxvp")
    pack = small_pack(pack_path)
    frames, starts = pack.flat_frames()
    rec["pack_frames"] = frames
    rec["pack_starts"] = starts
    rec["pack_counts"] = pack.frame_counts
    v = D.init_distractors("video", pack, key_from_seed(9), 40, env_offset=3)
    rec["video_init_seed9_off3_b40"] = v.video_index
    seq = [v.frame_cursor.copy()]
    dirs = [v.direction.copy()]
    for t in range(1, 14):
        v = D.advance_distractors(v, fold_in(key_from_seed(9), t), env_offset=3)
        seq.append(v.frame_cursor.copy())
        dirs.append(v.direction.copy())
    rec["video_cursor_seq"] = np.stack(seq)
    rec["video_dir_seq"] = np.stack(dirs)
    # composites on a random frame with a checker background mask
    rr = np.random.default_rng(3)
    fr = Frame.allocate(6, 24, 20)
    fr.pixels[:] = rr.integers(0, 256, fr.pixels.shape, dtype=np.uint8)
    yy, xx = np.meshgrid(np.arange(24), np.arange(20), indexing="ij")
    fr.depth[:] = np.where((yy + xx) % 3 == 0, 1.5, np.inf).astype(np.float32)
    rec["comp_pixels"] = fr.pixels.copy()
    rec["comp_depth"] = fr.depth.copy()
    cs = D.init_distractors("color", None, key_from_seed(1), 6)
    rec["comp_bias"] = cs.color_bias
    rec["comp_color_out"] = D.apply_color(fr, cs).pixels
    vs = D.init_distractors("video", pack, key_from_seed(2), 6)
    vs.frame_cursor[:] = [0, 1, 2, 3, 4, 2]
    rec["comp_vidx"] = vs.video_index
    rec["comp_cursor"] = vs.frame_cursor
    rec["comp_video_out"] = D.apply_video(fr, pack, vs).pixels
    np.savez_compressed(os.path.join(HERE, "distractor.npz"), **rec)


def replay_fixture(tag, model, batch, mode, steps, seed, observation="rgb",
                   env_offset=0, logical_batch=None, pack_path=None):
    """Reference env rollout: per-step poses / done flags / obs hash chain."""
    cfg = EnvConfig(model=MODELS[model], batch=batch, seed=seed, distractor_mode=mode,
                    video_pack_path=pack_path, observation=observation, threads=8,
                    env_offset=env_offset, logical_batch=logical_batch)
    env, state, obs = make_env(cfg)
    act = make_policy(f"random:{seed}", env)
    poses = [forward_kinematics(env.spec, state.sys.qpos)]
    dones = [np.zeros(batch, dtype=bool)]
    h = hashlib.sha256(b"\x00" * 32 + np.ascontiguousarray(obs).tobytes()).digest()
    hashes = [np.frombuffer(h, dtype=np.uint8)]
    first_obs = obs.copy()
    for t in range(steps):
        state, out = step(env, state, act(obs, t))
        obs = out.obs
        poses.append(forward_kinematics(env.spec, state.sys.qpos))
        dones.append(out.done.copy())
        h = hashlib.sha256(h + np.ascontiguousarray(obs).tobytes()).digest()
        hashes.append(np.frombuffer(h, dtype=np.uint8))
    rec = {
        "poses": np.stack(poses), "done": np.stack(dones), "hashes": np.stack(hashes),
        "first_obs": first_obs, "last_obs": obs,
        "meta": np.array(json.dumps({
            "model": model, "batch": batch, "mode": mode, "steps": steps, "seed": seed,
            "observation": observation, "env_offset": env_offset,
            "logical_batch": logical_batch if logical_batch is not None else batch,
            "floor_in_background": cfg.resolved_floor_in_background,
        })),
    }
    d = state.distractor
    rec["final_color_bias"] = d.color_bias
    rec["final_video_index"] = d.video_index
    rec["final_frame_cursor"] = d.frame_cursor
    rec["final_direction"] = d.direction
    if pack_path is not None:
        frames, starts = env.pack.flat_frames()
        rec["pack_frames"] = frames
        rec["pack_starts"] = starts
        rec["pack_counts"] = env.pack.frame_counts
    np.savez_compressed(os.path.join(HERE, f"replay_{tag}.npz"), **rec)
    print(tag, "resets:", int(np.stack(dones).sum()), "final", h.hex()[:16])


def physics_fixture():
    """One control step of the reference's step_dynamics + compute_reward
    (physics.py:427-477) from perturbed states, and reset_state draws
    (physics.py:487-510), for every model."""
    from pixelctrl.physics import SystemState, compute_reward, reset_state, step_dynamics

    rec = {}
    rng = np.random.default_rng(13)
    for name in MODELS:
        spec = spec_of(name)
        B = 32
        qpos = spec.rest()[None, :] + rng.uniform(-0.3, 0.3, (B, spec.dof))
        qpos[:, 1] = rng.uniform(0.2, 1.5, B)  # some envs in ground contact
        qvel = rng.normal(0.0, 0.5, (B, spec.dof))
        act = rng.uniform(-1.3, 1.3, (B, spec.n_joints))  # includes clamped values
        st = SystemState(qpos.copy(), qvel.copy(), rng.integers(0, 999, B).astype(np.int64),
                         np.zeros(B, dtype=bool))
        nxt = step_dynamics(spec, st, act)
        rec[f"{name}_qpos"] = qpos
        rec[f"{name}_qvel"] = qvel
        rec[f"{name}_steps"] = st.step_count
        rec[f"{name}_act"] = act
        rec[f"{name}_qpos1"] = nxt.qpos
        rec[f"{name}_qvel1"] = nxt.qvel
        rec[f"{name}_done1"] = nxt.done
        rec[f"{name}_reward"] = compute_reward(spec, st, nxt, act)
        rs = reset_state(spec, fold_in(key_from_seed(3), 0x5EED), 16, env_offset=5)
        rec[f"{name}_reset_qpos"] = rs.qpos
        rec[f"{name}_reset_qvel"] = rs.qvel
    np.savez_compressed(os.path.join(HERE, "physics.npz"), **rec)


def _scene_list():
    """Deterministic scenes for the generic render()/render_batch() API
    (render.py:491-552): random two-triangle scenes in the style of the
    reference's ray-cast acceptance test (tests/test_acceptance.py:158-188),
    posed sphere/capsule scenes under general cameras with and without the
    floor, and the 256x256 sphere of the silhouette test (190-199)."""
    rng = np.random.default_rng(7)
    scenes = []
    cam0 = Camera(eye=(0.0, -3.0, 0.5), target=(0.0, 1.0, 0.5))
    for _ in range(40):
        v = np.empty((6, 3), dtype=np.float32)
        v[:, 0] = rng.uniform(-2.0, 2.0, 6)
        v[:, 1] = rng.uniform(1.5, 6.0, 6)
        v[:, 2] = rng.uniform(-1.5, 3.0, 6)
        meshes = [(Mesh(v[3 * i:3 * i + 3].copy(), np.array([[0, 1, 2]], dtype=np.int32),
                        tuple(LINK_PALETTE[int(rng.integers(len(LINK_PALETTE)))])), Pose())
                  for i in range(2)]
        scenes.append((meshes, cam0, 32, 32, True))
    for k in range(12):
        meshes = []
        for j in range(int(rng.integers(1, 4))):
            if rng.random() < 0.5:
                m = tessellate_sphere(float(rng.uniform(0.2, 0.8)), int(rng.integers(3, 12)),
                                      int(rng.integers(4, 16)))
            else:
                m = tessellate_capsule(float(rng.uniform(0.05, 0.3)), float(rng.uniform(0.2, 1.2)),
                                       int(rng.integers(2, 6)), int(rng.integers(3, 12)),
                                       LINK_PALETTE[j % len(LINK_PALETTE)])
            pose = Pose(x=float(rng.uniform(-1, 1)), y=float(rng.uniform(-0.5, 0.5)),
                        z=float(rng.uniform(0.2, 1.5)), pitch=float(rng.uniform(-3, 3)))
            meshes.append((m, pose))
        eye = (float(rng.uniform(-2, 2)), float(rng.uniform(-5, -2)), float(rng.uniform(0.5, 3)))
        cam = Camera(eye=eye, target=(0.0, 0.0, 0.6), vertical_fov=float(rng.uniform(0.5, 1.2)))
        H, W = [(48, 64), (40, 40), (33, 57)][k % 3]
        scenes.append((meshes, cam, W, H, bool(k % 2)))
    sphere = tessellate_sphere(0.8, 32, 48)
    scenes.append(([(sphere, Pose(z=1.0))], Camera(eye=(0.0, -5.0, 1.0), target=(0.0, 0.0, 1.0)),
                   256, 256, True))
    scenes.append(([], cam0, 24, 16, False))  # empty scene: sky + floor only
    return scenes


def scene_fixture():
    rec = {"mesh_counts": [], "vert_counts": [], "tri_counts": [], "verts": [], "tris": [],
           "colors": [], "poses": [], "cams": [], "sizes": [], "fib": []}
    out_px, out_dp = [], []
    for meshes, cam, W, H, fib in _scene_list():
        rec["mesh_counts"].append(len(meshes))
        for m, pose in meshes:
            rec["vert_counts"].append(len(m.vertices))
            rec["tri_counts"].append(len(m.triangles))
            rec["verts"].append(np.asarray(m.vertices, np.float32))
            rec["tris"].append(np.asarray(m.triangles, np.int32))
            rec["colors"].append(np.asarray(m.base_color, np.float64))
            rec["poses"].append([pose.x, pose.y, pose.z, pose.pitch])
        rec["cams"].append(list(cam.eye) + list(cam.target) + list(cam.up) +
                           [cam.vertical_fov, cam.near, cam.far])
        rec["sizes"].append([H, W])
        rec["fib"].append(fib)
        fr = render(meshes, cam, width=W, height=H, floor_in_background=fib)
        out_px.append(fr.pixels[0].reshape(-1))
        out_dp.append(fr.depth[0].reshape(-1))
    arrs = {
        "mesh_counts": np.array(rec["mesh_counts"], np.int64),
        "vert_counts": np.array(rec["vert_counts"], np.int64),
        "tri_counts": np.array(rec["tri_counts"], np.int64),
        "verts": np.concatenate(rec["verts"]) if rec["verts"] else np.zeros((0, 3), np.float32),
        "tris": np.concatenate(rec["tris"]) if rec["tris"] else np.zeros((0, 3), np.int32),
        "colors": np.array(rec["colors"], np.float64),
        "poses": np.array(rec["poses"], np.float64),
        "cams": np.array(rec["cams"], np.float64),
        "sizes": np.array(rec["sizes"], np.int64),
        "fib": np.array(rec["fib"], bool),
        "pixels": np.concatenate(out_px),
        "depth": np.concatenate(out_dp),
    }
    # render_batch of three same-size scenes equals the singles (render.py:536-552)
    sc = [(m, c) for m, c, W, H, fib in _scene_list()[40:52] if (H, W) == (48, 64)][:3]
    fb = render_batch(sc, width=64, height=48, floor_in_background=False)
    arrs["batch_pixels"] = fb.pixels
    arrs["batch_depth"] = fb.depth
    np.savez_compressed(os.path.join(HERE, "scenes.npz"), **arrs)


def policy_fixture():
    """Conv-stub weights (a pure function of the seed) and the reference's
    own forward outputs (bench.py:36-145) for three shapes."""
    from pixelctrl.bench import ConvStub, conv_stub_forward

    rec = {}
    for tag, (h, w, c, j, seed, b) in {"a": (24, 28, 3, 5, 1, 3), "g": (16, 16, 1, 3, 2, 2),
                                       "f": (84, 84, 3, 17, 0, 4)}.items():
        stub = ConvStub.create(h, w, c, j, seed=seed)
        obs = np.random.default_rng(seed + 100).integers(0, 256, (b, h, w, c), dtype=np.uint8)
        rec[f"{tag}_shape"] = np.array([h, w, c, j, seed], np.int64)
        if tag == "f":  # large: only digests of the weights
            rec["f_weights_sha"] = np.array([sha(stub.conv), sha(stub.conv_blocks), sha(stub.proj)])
        else:
            rec[f"{tag}_conv"] = stub.conv
            rec[f"{tag}_conv_blocks"] = stub.conv_blocks
            rec[f"{tag}_proj"] = stub.proj
        rec[f"{tag}_obs"] = obs
        rec[f"{tag}_actions"] = conv_stub_forward(stub, obs)
    np.savez_compressed(os.path.join(HERE, "policy.npz"), **rec)


def recorder_fixture():
    """recorder.py: random-policy actions (a sliced batch), PNG bytes and
    a PXTJ digest file of a short rollout, all from the reference."""
    import tempfile

    from pixelctrl import recorder as R

    rec = {}
    cfg = EnvConfig(model="hopper_lite", batch=5, seed=2, env_offset=3, logical_batch=16)
    env, _, _ = make_env(cfg)
    for t in (0, 7):
        rec[f"random_actions_t{t}"] = R._random_actions(key_from_seed(5), t, env)
    img = np.random.default_rng(3).integers(0, 256, (13, 17, 3), dtype=np.uint8)
    rec["png_image"] = img
    with tempfile.TemporaryDirectory() as d:
        for tag, im in (("rgb", img), ("gray", img[..., 0])):
            path = os.path.join(d, f"{tag}.png")
            R.write_png(im, path)
            with open(path, "rb") as f:
                rec[f"png_{tag}_bytes"] = np.frombuffer(f.read(), dtype=np.uint8)
        dg = R.record_rollout(EnvConfig(model="hopper_lite", batch=2, seed=1), "zeros", 3)
        path = os.path.join(d, "d.pxtj")
        R.save_digest(dg, path)
        with open(path, "rb") as f:
            rec["digest_file"] = np.frombuffer(f.read(), dtype=np.uint8)
    np.savez_compressed(os.path.join(HERE, "recorder.npz"), **rec)


def main():
    if len(sys.argv) > 1 and sys.argv[1] == "recorder":
        recorder_fixture()
        return
    if len(sys.argv) > 1 and sys.argv[1] == "policy":
        policy_fixture()
        return
    if len(sys.argv) > 1 and sys.argv[1] == "physics":
        physics_fixture()
        return
    if len(sys.argv) > 1 and sys.argv[1] == "scenes":
        scene_fixture()
        return
    geometry_fixture()
    render_fixtures()
    distractor_fixtures()
    physics_fixture()
    scene_fixture()
    policy_fixture()
    recorder_fixture()
    pack = os.path.join("/tmp", "golden_replay.pxvp")
    small_pack(pack, seed=21, videos=4, frames=7, size=32)
    # BASELINE config 1: HalfCheetah, 1 env, 84x84, no distractors, 1000 steps.
    replay_fixture("cheetah_none_b1", "cheetah_lite", 1, "none", 1000, 0)
    replay_fixture("walker_video_b8", "walker_lite", 8, "video", 150, 1, pack_path=pack)
    replay_fixture("ant_color_b8", "ant_lite", 8, "color", 60, 2)
    replay_fixture("humanoid_video_b8_slice", "humanoid_lite", 8, "video", 120, 4,
                   env_offset=8, logical_batch=32, pack_path=pack)
    replay_fixture("hopper_color_gray_b4", "hopper_lite", 4, "color", 80, 5,
                   observation="grayscale")


if __name__ == "__main__":
    sys.exit(main())

"""Full-size oracle parity for every BASELINE configuration (-m gpu).

The fused step (distractor advance + auto-reset re-draw + render +
composite + grayscale, one pxr_render_step launch) is compared with the CPU
oracle on EVERY env of the batch, over several steps with real `done`
flags. At these sizes each CTA of the persistent grid renders many envs in
sequence, so this covers the cross-env machinery the small golden suites
cannot reach: the one-env-ahead prefetch of link trig and distractor slot,
the double-buffered link table, the video mbarrier parity flip, the TMA
store overlapping the next env, and (B > 32 x grid) the second and later
32-env distractor batches of a CTA.

Reference semantics followed (all under /root/reference/pkg/src/pixelctrl/):
render_robot_batch render.py:594-623; advance_distractors distractor.py:
116-137; video re-draw for done envs env.py:226-244; composites
distractor.py:140-214; grayscale env.py:168-173; big batch == slices
tests/test_acceptance.py:72-90, tests/test_env.py:168-206.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

# (bench model, envs, distractor mode, grayscale): BASELINE configs 2-5
CONFIGS = [
    ("Ant", 1024, "color", False),         # config 2 (floor instance, several envs per CTA)
    ("Walker2d", 4096, "video", False),    # config 3
    ("Humanoid", 4096, "video", False),    # config 4 (the headline)
    ("HalfCheetah", 16384, "none", False),  # config 5 sweep top cell, all four models
    ("Walker2d", 16384, "video", False),
    ("Ant", 16384, "color", False),
    ("Humanoid", 16384, "video", False),
    ("Walker2d", 4096, "video", True),     # grayscale composite
    ("Ant", 4096, "color", True),
]
# RGB video takes the pack upscaled to the frame size (one TMA copy per env);
# these run the per-pixel texel gather instead (PXR_DEBUG_NO_UPSCALE)
GATHER = [("Humanoid", 4096, "video", False), ("Walker2d", 16384, "video", False)]
CASES = [c + (False,) for c in CONFIGS] + [c + (True,) for c in GATHER]

STEPS = 3
DONE_RATE = 0.15


def _oracle_step(oracle, w, hp, st, frames, starts):
    px, dp = oracle.render_robot_batch(w.geom, hp, w.width, w.height, w.floor_in_background,
                                       threads=oracle.host_threads())
    if w.mode == "color":
        oracle.apply_color_inplace(px, st["color_bias"], threads=oracle.host_threads())
    elif w.mode == "video":
        oracle.apply_video_inplace(px, dp, frames, starts[st["video_index"]] + st["frame_cursor"],
                                   threads=oracle.host_threads())
    return (oracle.grayscale(px) if w.grayscale else px), dp


def _check_state(w, st):
    got = w.dist.to_host()
    for k, v in st.items():
        np.testing.assert_array_equal(got[k], v, err_msg=k)


def _first_bad_env(a, b):
    bad = np.nonzero((a != b).reshape(a.shape[0], -1).any(axis=1))[0]
    return bad[:10]


@pytest.mark.parametrize("model,B,mode,gray,gather", CASES,
                         ids=[f"{m}-{b}-{d}{'-gray' if g else ''}{'-gather' if q else ''}"
                              for m, b, d, g, q in CASES])
def test_fused_step_full_batch(torch, pkg, oracle, knobs, model, B, mode, gray, gather):
    from paper_2502_00021_b200 import bench_support as bs

    if gather:
        knobs.set("PXR_DEBUG_NO_UPSCALE", 1)

    seed = 11
    w = bs.Workload(model, B, mode, seed=seed, grayscale=gray)
    frames = starts = counts = None
    if w.pack is not None:
        frames, starts = w.pack.flat_frames()
        counts = np.asarray(w.pack.frame_counts, dtype=np.int64)
    master = oracle.key_from_seed(seed)
    st = oracle.init_distractors(mode, counts, oracle.fold_in(master, 0xD157), B)
    _check_state(w, st)  # the device init (pxr_init_distractors) over the whole batch
    rng = np.random.default_rng(B + len(model))
    for t in range(STEPS):
        done = rng.random(B) < DONE_RATE
        done_dev = torch.from_numpy(done.astype(np.uint8)).cuda()
        poses = w.poses(t)
        obs, _ = w.render(poses, t, done=done_dev, want_depth=False)  # the production path
        torch.cuda.synchronize()
        st = oracle.advance_state(st, mode, oracle.fold_in(master, t), 0, B,
                                  frame_counts=counts, done=done)
        _check_state(w, st)
        want, dp = _oracle_step(oracle, w, poses.cpu().numpy(), st, frames, starts)
        got = obs.cpu().numpy()
        assert np.array_equal(got, want), (
            f"t={t}: envs {_first_bad_env(got, want)} differ from the oracle")
    # the observe() path (no advance) with the depth output: same obs, exact depth
    obs2, depth = w.render(poses, STEPS - 1, advance=False, want_depth=True,
                           out_obs=torch.empty_like(w.obs))
    torch.cuda.synchronize()
    assert np.array_equal(obs2.cpu().numpy(), want)
    assert np.array_equal(depth.cpu().numpy().view(np.uint32), dp.view(np.uint32))


def test_device_pose_source_matches_host(torch, pkg, oracle):
    """The bench's on-device pose source vs its host restatement (the
    reference arm's poses): bit-identical (glibc sin on both sides)."""
    from paper_2502_00021_b200 import bench_support as bs
    from paper_2502_00021_b200.models import model_kinematics

    for model in ("HalfCheetah", "Walker2d", "Ant", "Humanoid"):
        w = bs.Workload(model, 2048, "none", seed=0, env_offset=512)
        par, anc, _, _ = model_kinematics(w.spec)
        rk = (w.reset_key.hi, w.reset_key.lo)
        for t in (0, 17):
            dev = w.poses(t).cpu().numpy()
            host = oracle.pose_source(w.spec.rest(), par, anc, rk, 512, t, 2048)
            np.testing.assert_array_equal(dev, host)

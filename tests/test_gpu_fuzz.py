"""Seeded randomized parity of the fused kernel against the C oracle: random
model, distractor mode, frame size (8..139 per side, some forced into row
bands), camera offset / field of view, floor on/off, grayscale, large-angle
poses, and a video pack of odd size (so both the byte-permute gather and the
generic texel path run). Pixels, depth and the distractor composite must be
bit-exact for every case."""

import os

import numpy as np
import pytest

from conftest import MODEL_NAMES, geometry_of, spec_of

pytestmark = pytest.mark.gpu


def _case(seed):
    rng = np.random.default_rng(7000 + seed)
    name = MODEL_NAMES[int(rng.integers(len(MODEL_NAMES)))]
    mode = ("none", "color", "video")[int(rng.integers(3))]
    H, W = (int(v) for v in rng.integers(8, 140, 2))
    band = int(rng.integers(3, max(4, H))) if rng.random() < 0.3 else 0
    offset = (float(rng.uniform(-1.0, 1.0)), float(rng.uniform(-5.0, -2.0)),
              float(rng.uniform(0.4, 2.5)))
    fov = float(rng.uniform(0.6, 1.3))
    fib = bool(rng.random() < 0.5)
    gray = bool(rng.random() < 0.3)
    hv, wv = (int(v) for v in rng.integers(9, 70, 2))
    return rng, name, mode, H, W, band, offset, fov, fib, gray, hv, wv


# PXR_FUZZ_SEEDS=N widens the sweep for soak runs (default 40)
# + seeds a 2000-seed soak found (RGB video WITH the floor drawn: the upscaled
# frame copy must not replace the floor background)
REGRESSION_SEEDS = (78, 301, 411, 1927)


@pytest.mark.parametrize("seed", sorted(set(range(int(os.environ.get("PXR_FUZZ_SEEDS", "40"))))
                                        | set(REGRESSION_SEEDS)))
def test_fused_render_fuzz_vs_oracle(pkg, torch, oracle, knobs, seed):
    rng, name, mode, H, W, band, offset, fov, fib, gray, hv, wv = _case(seed)
    # one env per CTA, or 1-3 CTAs rendering several envs each
    if seed % 4:
        knobs.set("PXR_DEBUG_GRID", seed % 4)
    if band:
        knobs.set("PXR_DEBUG_BAND_H", str(band))
    from paper_2502_00021_b200.models import forward_kinematics_host

    spec = spec_of(name)
    geom = geometry_of(name)
    B = 12
    qpos = np.tile(spec.rest(), (B, 1))
    qpos[:, 0] += rng.uniform(-2.0, 2.0, B)
    qpos[:, 1] += rng.uniform(-0.3, 0.6, B)
    qpos[:, 2:] += rng.uniform(-np.pi, np.pi, (B, spec.dof - 2))
    poses = forward_kinematics_host(spec, qpos)
    pack = dpack = None
    if mode == "video":
        vids = [rng.integers(0, 256, (int(rng.integers(2, 6)), hv, wv, 3), dtype=np.uint8)
                for _ in range(3)]
        pack = pkg.VideoPack(videos=vids, height=hv, width=wv)
        dpack = pack.to_device()
    dist = pkg.init_distractors(mode, pack, pkg.key_from_seed(seed), B)
    cfg = pkg.CameraConfig(offset=offset, vertical_fov=fov)
    r = pkg.RobotRenderer(geom, cfg, W, H)
    obs, depth = r.render(torch.from_numpy(poses).cuda(), floor_in_background=fib, dist=dist,
                          pack=dpack, grayscale=gray, want_depth=True)
    px, dp = oracle.render_robot_batch(geom, poses, W, H, fib, threads=4, offset=offset,
                                       fov=fov)
    tag = f"seed {seed}: {name} {mode} {H}x{W} band={band} fib={fib} gray={gray}"
    np.testing.assert_array_equal(depth.cpu().numpy().view(np.uint32), dp.view(np.uint32),
                                  err_msg=tag)
    host = dist.to_host()
    if mode == "color":
        oracle.apply_color_inplace(px, host["color_bias"])
    elif mode == "video":
        frames, starts = pack.flat_frames()
        oracle.apply_video_inplace(px, dp, frames, starts[host["video_index"]] +
                                   host["frame_cursor"])
    if gray:
        px = oracle.grayscale(px)
    np.testing.assert_array_equal(obs.cpu().numpy(), px, err_msg=tag)

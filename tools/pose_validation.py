"""Is the bench's on-device pose source representative? (SURVEY.md 8(d):
its render workload must be within +-20 % of reference-physics rollouts.)

For each model: reference-physics poses (the recorded reference rollouts,
tests/golden/replay_*.npz: physics.py:487-510 + env.py:201-255 under the
random policy) against the pose source (pxr_pose_source: reference reset
keys + joint oscillation + FK) over 4096 envs and several steps. Both are
rendered WITHOUT the floor, with the per-env workload counters of the
checked build (PXR_DEBUG_STATS_PTR): foreground pixels (finite depth),
live triangles, bbox-row units, candidate pixels. Prints a markdown table."""
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "tests"))
os.environ.setdefault("PXR_LIB_PATH", os.path.join(REPO, "paper_2502_00021_b200",
                                                   "libpxr_checked.so"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from conftest import golden  # noqa: E402
from paper_2502_00021_b200 import _native  # noqa: E402
from paper_2502_00021_b200.bench_support import Workload  # noqa: E402

REPLAYS = {"cheetah_lite": ("cheetah_none_b1", "HalfCheetah"),
           "walker_lite": ("walker_video_b8", "Walker2d"),
           "ant_lite": ("ant_color_b8", "Ant"),
           "humanoid_lite": ("humanoid_video_b8_slice", "Humanoid"),
           "hopper_lite": ("hopper_color_gray_b4", "hopper_lite")}
STEPS = (0, 25, 50, 100, 200, 400)


def measure(renderer, poses):
    B = poses.shape[0]
    stats = torch.full((B, 11), -1, dtype=torch.int32, device="cuda")  # kStats
    _native.set_debug("PXR_DEBUG_STATS_PTR", stats.data_ptr())
    _, depth = renderer.render(poses, floor_in_background=True, want_depth=True)
    torch.cuda.synchronize()
    _native.set_debug("PXR_DEBUG_STATS_PTR", None)
    st = stats.cpu().numpy().astype(np.float64)
    assert (st >= 0).all()
    fg = torch.isfinite(depth).float().mean(dim=(1, 2)).cpu().numpy()
    return {"fg_pct": 100 * fg.mean(), "live": st[:, 0].mean(), "rows": st[:, 1].mean(),
            "cand": st[:, 3].mean()}


rows = []
for name, (tag, bench) in REPLAYS.items():
    ref = golden(f"replay_{tag}.npz")["poses"]
    ref = ref.reshape(-1, ref.shape[2], 3)
    w = Workload(bench, 4096, "none")
    a = measure(w.renderer, torch.from_numpy(np.ascontiguousarray(ref)).cuda())
    src = [measure(w.renderer, w.poses(t).clone()) for t in STEPS]
    b = {k: float(np.mean([s[k] for s in src])) for k in a}
    rows.append((name, len(ref), a, b))

print("| model | reference poses | fg px % ref / source | live tris ref / source | "
      "bbox-row units ref / source | candidates ref / source | worst deviation |")
print("|---|---|---|---|---|---|---|")
for name, n, a, b in rows:
    dev = max(abs(b[k] / a[k] - 1) for k in a)
    print(f"| {name} | {n} | {a['fg_pct']:.2f} / {b['fg_pct']:.2f} | {a['live']:.0f} / {b['live']:.0f} "
          f"| {a['rows']:.0f} / {b['rows']:.0f} | {a['cand']:.0f} / {b['cand']:.0f} | {100 * dev:+.1f} % |")

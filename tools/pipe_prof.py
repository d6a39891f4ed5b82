"""Stage cycle counters of the warp-specialised render pipeline
(pxr_render_pipe.cu, PXR_DEBUG_PIPE_PROF): per CTA, where the geometry
warps (G) and the raster warps (R) spend their cycles, averaged over the
CTAs; plus the device time of the same launch with both render kernels."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2502_00021_b200 import _native  # noqa: E402
from paper_2502_00021_b200.bench_support import Workload  # noqa: E402

SLOTS = {0: "G wait env buffers", 1: "G prepare (trig, distractor)", 2: "G vertex",
         3: "G liveness + scan", 4: "G wait round buffer", 5: "G records",
         6: "G total", 8: "R wait records", 9: "R env init", 10: "R raster",
         11: "R final pass", 12: "R total", 13: "rounds", 14: "envs"}

ap = argparse.ArgumentParser()
ap.add_argument("--model", default="Humanoid")
ap.add_argument("--envs", type=int, default=4096)
ap.add_argument("--mode", default="video")
ap.add_argument("--timed", type=int, default=50)
a = ap.parse_args()
w = Workload(a.model, a.envs, a.mode)
poses = [w.poses(t).clone() for t in range(2)]


def timed(variant):
    _native.set_debug("PXR_DEBUG_RENDER", variant)
    for t in range(4):
        w.render(poses[t % 2], t)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record()
    for t in range(a.timed):
        w.render(poses[t % 2], 4 + t)
    ev[1].record()
    torch.cuda.synchronize()
    return ev[0].elapsed_time(ev[1]) / a.timed


for v in ("legacy", "pipe", "legacy", "pipe"):
    ms = timed(v)
    print(f"{a.model} {a.mode} B={a.envs} {v}: {ms:.4f} ms  {a.envs / ms / 1e3:.2f} M env-steps/s")
_native.set_debug("PXR_DEBUG_RENDER", "pipe")
prof = torch.zeros((1024, 16), dtype=torch.int64, device="cuda")
_native.set_debug("PXR_DEBUG_PIPE_PROF", prof.data_ptr())
w.render(poses[0], 100)
torch.cuda.synchronize()
_native.set_debug("PXR_DEBUG_PIPE_PROF", None)
P = prof.cpu().numpy()
P = P[P[:, 14] > 0]
print(f"CTAs {len(P)}, envs/CTA {P[:, 14].mean():.1f}, rounds/env {P[:, 13].sum() / P[:, 14].sum():.3f}")
for s, name in SLOTS.items():
    if s in (13, 14):
        continue
    print(f"  {name:32s} {P[:, s].mean() / 1965:9.2f} us  ({P[:, s].mean() / P[:, 14].mean():9.0f} cyc/env)")

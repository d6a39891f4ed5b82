"""Profiling driver: set up one bench workload and run fused steps (no soak,
no CPU legs) so ncu can capture the render kernel in isolation; prints the
mean device time of the last --timed launches."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2502_00021_b200.bench_support import Workload  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--model", default="Humanoid")
ap.add_argument("--envs", type=int, default=4096)
ap.add_argument("--mode", default="video")
ap.add_argument("--steps", type=int, default=4)
ap.add_argument("--timed", type=int, default=20)
ap.add_argument("--grayscale", action="store_true")
ap.add_argument("--size", type=int, nargs=2, default=(84, 84), metavar=("H", "W"))
a = ap.parse_args()
w = Workload(a.model, a.envs, a.mode, grayscale=a.grayscale, height=a.size[0], width=a.size[1])
poses = [w.poses(t).clone() for t in range(2)]
torch.cuda.synchronize()
for t in range(a.steps):
    w.render(poses[t % 2], t)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ev[0].record()
for t in range(a.timed):
    w.render(poses[t % 2], a.steps + t)
ev[1].record()
torch.cuda.synchronize()
ms = ev[0].elapsed_time(ev[1]) / max(1, a.timed)
print(f"{a.model} {a.mode} {a.size[0]}x{a.size[1]} B={a.envs}: {ms:.3f} ms/launch  {a.envs / ms / 1e3:.2f} M env-steps/s")

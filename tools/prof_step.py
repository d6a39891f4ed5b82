"""Profiling driver: set up one bench workload and run a few fused steps
(no soak, no CPU legs) so ncu can capture the render kernel in isolation."""
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
ap.add_argument("--steps", type=int, default=6)
ap.add_argument("--grayscale", action="store_true")
a = ap.parse_args()
w = Workload(a.model, a.envs, a.mode, grayscale=a.grayscale)
poses = [w.poses(t).clone() for t in range(2)]
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
for t in range(a.steps):
    if t == a.steps - 1:
        ev[0].record()
    w.render(poses[t % 2], t)
    if t == a.steps - 1:
        ev[1].record()
torch.cuda.synchronize()
print(f"{a.model} {a.mode} B={a.envs}: last launch {ev[0].elapsed_time(ev[1]):.3f} ms")

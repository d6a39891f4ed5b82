"""Per-phase cycles of the fused render kernel (debug hook
PXR_DEBUG_PROF: thread 0's clock at each phase-ending barrier, per CTA),
averaged per env, plus the launch's device time with the host out of the
loop (20 launches captured in one CUDA graph and replayed). Loads
libpxr_prof.so (the timers are compiled out of libpxr.so) unless
PXR_LIB_PATH names another build."""
import argparse
import os
import sys

os.environ.setdefault("PXR_LIB_PATH", os.path.join(
    os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2502_00021_b200",
    "libpxr_prof.so"))

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2502_00021_b200 import _native  # noqa: E402
from paper_2502_00021_b200.bench_support import Workload  # noqa: E402

SLOTS = ["setup + first prepare", "vertex", "liveness + scan", "records (+bg)", "raster",
         "resolve", "paint + store issue", "final store wait"]

ap = argparse.ArgumentParser()
ap.add_argument("--cases", nargs="+", default=["HalfCheetah:none:1", "Humanoid:video:1",
                                               "HalfCheetah:none:100", "Humanoid:video:4096"])
a = ap.parse_args()
for case in a.cases:
    model, mode, B = case.split(":")
    B = int(B)
    w = Workload(model, B, mode)
    poses = w.poses(3).clone()
    for t in range(3):
        w.render(poses, t)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            for t in range(20):
                w.render(poses, 10 + t, stream=s)
    torch.cuda.current_stream().wait_stream(s)
    g.replay()
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record()
    for _ in range(10):
        g.replay()
    ev[1].record()
    torch.cuda.synchronize()
    us = ev[0].elapsed_time(ev[1]) / 200 * 1e3
    prof = torch.zeros((1024, 12), dtype=torch.int64, device="cuda")
    _native.set_debug("PXR_DEBUG_PROF", prof.data_ptr())
    w.render(poses, 99)
    torch.cuda.synchronize()
    _native.set_debug("PXR_DEBUG_PROF", None)
    P = prof.cpu().numpy()
    P = P[P[:, 8] > 0]
    envs = P[:, 8].sum()
    print(f"{model} {mode} B={B}: {us:.2f} us/launch (graph replay), {len(P)} CTAs, "
          f"{envs / len(P):.1f} envs/CTA")
    tot = P[:, :8].sum(axis=1).mean()
    for i, n in enumerate(SLOTS):
        c = P[:, i].mean()
        print(f"   {n:24s} {c / 1965:8.2f} us/CTA  {c / (envs / len(P)):8.0f} cyc/env  {100 * c / tot:5.1f} %")
    per = envs / len(P)
    print(f"   raster detail per env: rows drawn {P[:, 10].mean() / per:6.0f} cyc, pool "
          f"evaluated {P[:, 11].mean() / per:6.0f} cyc, next-env preparation (1 warp) "
          f"{P[:, 9].mean() / per:6.0f} cyc")

"""Device time per render launch with and without a debug knob (default
PXR_DEBUG_NO_PDL: programmatic dependent launch; PXR_DEBUG_NO_SPLIT: small
batches split over CTAs), same library, interleaved: host launch loop and a
CUDA graph of 20 launches, small batches (BASELINE config 1, the sweep's
{1, 10, 100} cells) and the 4096-env headline.
usage: python tools/pdl_ab.py [KNOB] [--small]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2502_00021_b200 import _native  # noqa: E402
from paper_2502_00021_b200.bench_support import Workload  # noqa: E402


def timed(fn, n):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record()
    for _ in range(n):
        fn()
    ev[1].record()
    torch.cuda.synchronize()
    return ev[0].elapsed_time(ev[1]) / n * 1e3  # us


KNOB = next((a for a in sys.argv[1:] if a.startswith("PXR_")), "PXR_DEBUG_NO_PDL")
SMALL = "--small" in sys.argv


def run(model, mode, B, pdl, two=False):
    _native.set_debug(KNOB, None if pdl else "1")
    w = Workload(model, B, mode)
    poses = w.poses(3).clone()
    s = torch.cuda.Stream()
    t = [0]

    def step():
        t[0] += 1
        if two:  # pose-source kernel + render (Workload.step)
            w.step(t[0])
        else:
            w.render(poses, t[0], stream=s)
    with torch.cuda.stream(s):
        loop = timed(step, 200 if B < 1000 else 50)
        step()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(20):
                step()
        gr = timed(g.replay, 30 if B < 1000 else 5) / 20
    _native.set_debug(KNOB, None)
    return loop, gr


CASES = (("HalfCheetah", "none", 1), ("Humanoid", "video", 1), ("HalfCheetah", "none", 10),
         ("Humanoid", "video", 100), ("Humanoid", "video", 4096), ("Ant", "color", 1024))
if SMALL:
    CASES = (("HalfCheetah", "none", 1), ("Humanoid", "none", 1), ("Ant", "color", 1),
             ("HalfCheetah", "none", 10), ("Walker2d", "color", 10), ("Ant", "color", 64),
             ("Humanoid", "video", 1), ("Humanoid", "none", 100))
for model, mode, B in CASES:
    for rep in range(2):
        for pdl in (False, True):
            loop, gr = run(model, mode, B, pdl)
            print(f"{model:12s} {mode:6s} B={B:5d} {KNOB[11:].lower()}={int(not pdl)}: host loop {loop:8.2f} us, "
                  f"graph {gr:8.2f} us per launch", flush=True)
for model, mode, B in (("HalfCheetah", "none", 1), ("Humanoid", "video", 4096)) if not SMALL else ():
    for rep in range(2):
        for pdl in (False, True):
            loop, gr = run(model, mode, B, pdl, two=True)
            print(f"{model:12s} {mode:6s} B={B:5d} {KNOB[11:].lower()}={int(not pdl)}: pose source + render: host loop "
                  f"{loop:8.2f} us, graph {gr:8.2f} us per step", flush=True)

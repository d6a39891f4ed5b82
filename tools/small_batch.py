"""Device time per fused render launch at small batches (the latency-bound
end of the sweep: BASELINE config 1 and the {1, 10, 100} cells), next to
an empty-kernel launch on the same stream for the launch floor."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2502_00021_b200.bench_support import Workload  # noqa: E402


def timed(fn, n=300):
    for _ in range(10):
        fn()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record()
    for _ in range(n):
        fn()
    ev[1].record()
    torch.cuda.synchronize()
    return ev[0].elapsed_time(ev[1]) / n * 1e3  # us


x = torch.zeros(1, device="cuda")
print(f"empty launch (x.add_(0)): {timed(lambda: x.add_(0)):.2f} us")
for model, mode in (("HalfCheetah", "none"), ("Humanoid", "video"), ("Ant", "color"),
                    ("Walker2d", "video")):
    for B in (1, 10, 100):
        w = Workload(model, B, mode)
        poses = w.poses(3).clone()
        t = [0]

        def step():
            t[0] += 1
            w.render(poses, t[0])
        print(f"{model:12s} {mode:6s} B={B:4d}: {timed(step):7.2f} us/launch")

"""Conv-stub policy timing (pxr_conv_stub_forward: tensor-core convolution +
projection) over batch sizes, device-timed; under ncu it gives the two
kernels' split."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2502_00021_b200.bench import ConvStub, conv_stub_forward  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--batches", type=int, nargs="+", default=[1, 100, 1000, 4096, 16384])
ap.add_argument("--joints", type=int, default=17)
ap.add_argument("--iters", type=int, default=20)
a = ap.parse_args()
stub = ConvStub.create(84, 84, 3, a.joints, seed=0)
for B in a.batches:
    obs = torch.randint(0, 256, (B, 84, 84, 3), dtype=torch.uint8, device="cuda")
    for _ in range(3):
        conv_stub_forward(stub, obs)
    e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    torch.cuda.synchronize()
    e[0].record()
    for _ in range(a.iters):
        conv_stub_forward(stub, obs)
    e[1].record()
    torch.cuda.synchronize()
    ms = e[0].elapsed_time(e[1]) / a.iters
    print(f"policy B={B} J={a.joints}: {ms:.3f} ms  ({B / ms / 1e3:.2f} M env/s)", flush=True)

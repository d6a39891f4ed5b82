"""Per-env workload counters of the fused render kernel (debug hook
PXR_DEBUG_STATS_PTR, csrc/pxr_render.cu kStats; checked build only): live triangles, bbox-row
units, non-empty row spans, candidate pixels, covered fragments, raster
rounds and fragment-list overflows, summarised over one step of a bench
workload. Used to size the kernel's per-round budgets and to aim
optimisations; not part of any timed path."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

# the counters are compiled into the checked build only
os.environ.setdefault("PXR_LIB_PATH", os.path.join(os.path.dirname(os.path.dirname(
    os.path.abspath(__file__))), "paper_2502_00021_b200", "libpxr_checked.so"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2502_00021_b200.bench_support import Workload  # noqa: E402

NAMES = ("live_tris", "row_units", "spans", "candidates", "fragments", "rounds", "overflows",
         "live_uncovering", "their_units", "their_1row", "trimmed_rows")

ap = argparse.ArgumentParser()
ap.add_argument("--model", default="Humanoid")
ap.add_argument("--envs", type=int, default=4096)
ap.add_argument("--mode", default="video")
ap.add_argument("--step", type=int, default=3)
ap.add_argument("--size", type=int, nargs=2, default=(84, 84), metavar=("H", "W"))
a = ap.parse_args()
from paper_2502_00021_b200 import _native
w = Workload(a.model, a.envs, a.mode, height=a.size[0], width=a.size[1])
stats = torch.full((a.envs, len(NAMES)), -1, dtype=torch.int32, device="cuda")
_native.set_debug("PXR_DEBUG_STATS_PTR", stats.data_ptr())
w.render(w.poses(a.step), a.step)
torch.cuda.synchronize()
_native.set_debug("PXR_DEBUG_STATS_PTR", None)
st = stats.cpu().numpy()
assert (st >= 0).all(), "stats not written for every env"
print(f"{a.model} {a.mode} {a.size[0]}x{a.size[1]} B={a.envs} step {a.step}")
print(f"{'counter':>11} {'mean':>9} {'p50':>7} {'p99':>7} {'max':>7}")
for i, n in enumerate(NAMES):
    c = st[:, i].astype(np.float64)
    print(f"{n:>11} {c.mean():9.1f} {np.percentile(c, 50):7.0f} {np.percentile(c, 99):7.0f} "
          f"{c.max():7.0f}")

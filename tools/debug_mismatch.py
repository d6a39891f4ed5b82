"""Debug helper: render a golden fixture on the GPU and dump mismatches."""
import os, sys, json
import numpy as np
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO); sys.path.insert(0, os.path.join(REPO, "tests"))
import torch
from conftest import golden, geometry_of
import paper_2502_00021_b200 as P
name = sys.argv[1] if len(sys.argv) > 1 else "cheetah_lite"
rec = golden(f"render_{name}.npz")
geom = geometry_of(name)
fr = P.render_robot_batch(geom, torch.from_numpy(rec["poses"]).cuda(), P.CameraConfig(), 84, 84, False)
px = fr.pixels.cpu().numpy(); dp = fr.depth.cpu().numpy()
want = rec["pixels_fib0"]; wd = rec["depth_fib0"]
bad = np.argwhere(np.any(px != want, axis=-1))
print("mismatched px", len(bad), "depth mismatches", int((dp.view(np.uint32) != wd.view(np.uint32)).sum()))
out = []
for b, y, x in bad[:40]:
    out.append([int(b), int(y), int(x), px[b, y, x].tolist(), want[b, y, x].tolist(), float(dp[b, y, x]), float(wd[b, y, x])])
print(json.dumps(out))
bb = np.unique(bad[:, 0]); print("envs", bb.tolist()[:50])

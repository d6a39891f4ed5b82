"""Wall time of the generic scene API's render_batch (reference
render.py:536-552) for a batch of random posed-capsule scenes, against a
loop of single render() calls."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2502_00021_b200 as P  # noqa: E402

rng = np.random.default_rng(0)
scenes = []
for i in range(64):
    meshes = [(P.tessellate_capsule(0.05 + 0.05 * rng.random(), 0.3 + 0.4 * rng.random()),
               P.Pose(rng.uniform(-1, 1), rng.uniform(-0.5, 0.5), rng.uniform(0.2, 1.0),
                      rng.uniform(-3, 3))) for _ in range(6)]
    cam = P.track_camera((rng.uniform(-1, 1), rng.uniform(0, 1)))
    scenes.append((meshes, cam))
for name, fn in (("render_batch", lambda: P.render_batch(scenes, 84, 84)),
                 ("render x64", lambda: [P.render(m, c, width=84, height=84) for m, c in scenes])):
    fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    print(f"{name}: {(time.perf_counter() - t) / 5 * 1e3:.2f} ms for 64 scenes")
a = P.render_batch(scenes, 84, 84)
for i in (0, 17, 63):
    b = P.render(scenes[i][0], scenes[i][1], width=84, height=84)
    assert torch.equal(a.pixels[i], b.pixels[0]) and torch.equal(a.depth[i], b.depth[0])
print("render_batch == singles")

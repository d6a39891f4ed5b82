"""The parity suites again, through the checked build (libpxr_checked.so,
-DPXR_CHECKED): every shared-memory index of the fused render kernel (record,
span, row-owner, candidate-pool, fragment and pixel slots, the video texel and
byte-permute reads), the distractor / frame indices, the policy kernel's
im2col and operand writes and the physics kernel's tree invariants are
checked on the device, and a failed check traps the launch. Run in a child
pytest with PXR_LIB_PATH pointing at the checked library, so a trap cannot
poison this process's CUDA context; the child asserts it really loaded the
checked build. This stands in for a memory checker (not available on the GPU
pool): the fuzz cases, the forced multi-round / fragment-overflow / row-band
paths and the env loop all run with the checks on and must stay bit-exact."""

import os
import re
import subprocess
import sys

import pytest

from conftest import REPO

pytestmark = pytest.mark.gpu

CHECKED = os.path.join(REPO, "paper_2502_00021_b200", "libpxr_checked.so")
SUITES = ["tests/test_gpu_fuzz.py", "tests/test_gpu_parity.py", "tests/test_policy.py",
          "tests/test_physics_api.py", "tests/test_env_gpu.py", "tests/test_scenes.py",
          "tests/test_gpu_determinism.py", "tests/test_gpu_render_api.py",
          "tests/test_gpu_distractor_api.py", "tests/test_gpu_env_api.py",
          "tests/test_gpu_physics_props.py", "tests/test_recorder_api.py"]


def test_parity_suites_under_device_checks():
    assert os.path.exists(CHECKED), "build it: make -C paper_2502_00021_b200/csrc checked"
    env = dict(os.environ, PXR_LIB_PATH=CHECKED, PXR_EXPECT_CHECKED="1")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu",
                        "-p", "no:cacheprovider", *SUITES],
                       cwd=REPO, env=env, capture_output=True, text=True, timeout=1500)
    out = r.stdout + r.stderr
    assert "PXR_DCHECK failed" not in out, out[-4000:]
    assert r.returncode == 0, out[-4000:]
    assert "checked build loaded" in out, out[-2000:]
    m = re.search(r"(\d+) passed", out)
    assert m and int(m.group(1)) >= 80, out[-2000:]  # the suites really ran
    print(out.strip().splitlines()[-1])


_BAD_LINK = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
import paper_2502_00021_b200 as P
from paper_2502_00021_b200 import _native
assert _native.lib().pxr_build_checked() == 1
geom = P.RobotGeometry([0.5, 0.4], [0.05, 0.04])
r = P.RobotRenderer(geom, P.CameraConfig(), 32, 32)
t, _ = geom.device_arrays(r.device)
t["vert_link"][5] = 7  # beyond n_links: the kernel would read another env's trig
poses = torch.zeros((4, 2, 3), dtype=torch.float64, device="cuda")
poses[:, :, 1] = 0.6
try:
    r.render(poses, floor_in_background=False)
    torch.cuda.synchronize()
except Exception as e:
    print("launch failed:", type(e).__name__)
    sys.exit(3)
print("no failure")
"""


def test_a_failed_check_traps_the_launch():
    """Negative control: a corrupted link index in device memory (something
    the host cannot validate) must stop the checked kernel, not render."""
    env = dict(os.environ, PXR_LIB_PATH=CHECKED)
    r = subprocess.run([sys.executable, "-c", _BAD_LINK, REPO], cwd=REPO, env=env,
                       capture_output=True, text=True, timeout=300)
    out = r.stdout + r.stderr
    assert r.returncode == 3 and "launch failed" in out, out[-3000:]
    assert "PXR_DCHECK failed" in out and "p.nl" in out, out[-3000:]


_STATS = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
from paper_2502_00021_b200 import _native
from paper_2502_00021_b200.bench_support import Workload
assert _native.lib().pxr_build_checked() == 1
K = 11  # csrc/pxr_render.cu kStats
for model, mode, B, knob in (("Humanoid", "video", 300, None), ("Ant", "color", 300, None),
                             ("HalfCheetah", "none", 40, "PXR_DEBUG_GRID"), ("Walker2d", "color", 5, None)):
    if knob:
        _native.set_debug(knob, 3)
    w = Workload(model, B, mode)
    st = torch.full((B, K), -1, dtype=torch.int32, device="cuda")
    _native.set_debug("PXR_DEBUG_STATS_PTR", st.data_ptr())
    w.render(w.poses(3), 3)
    torch.cuda.synchronize()
    _native.set_debug("PXR_DEBUG_STATS_PTR", None)
    if knob:
        _native.set_debug(knob, None)
    s = st.cpu().numpy().astype(np.int64)
    assert (s >= 0).all(), (model, "counters not written for every env")
    live, units, spans, cand, frags, rounds, over, unc, unc_units, unc_1, trim = s.T
    assert (over == 0).all(), model
    if B * 2 > 148:  # one band per env (the split launch counts its last band only)
        assert (live > 0).all() and (rounds >= 1).all(), model
    assert (units >= live).all() and (spans <= units).all() and (trim <= units).all(), model
    assert (cand >= spans).all() and (frags <= cand).all() and (unc <= live).all(), model
    assert (unc_1 <= unc).all() and (unc_units >= unc).all(), model
    print(model, mode, B, "live", live.mean(), "units", units.mean(), "cand", cand.mean())
print("stats ok")
"""


def test_workload_counters_consistent():
    """The checked build's per-env workload counters (tools/render_stats.py)
    on the one-CTA-per-env, several-envs-per-CTA and split launches: written
    for every env (a split env: its last band's counters) and mutually
    consistent (live triangles <= bbox-row units,
    spans <= units, candidates >= spans, fragments <= candidates, no
    fragment-list overflow at the default budgets)."""
    env = dict(os.environ, PXR_LIB_PATH=CHECKED)
    r = subprocess.run([sys.executable, "-c", _STATS, REPO], cwd=REPO, env=env,
                       capture_output=True, text=True, timeout=300)
    out = r.stdout + r.stderr
    assert r.returncode == 0 and "stats ok" in out, out[-3000:]
    assert "PXR_DCHECK failed" not in out, out[-3000:]

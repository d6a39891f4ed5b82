"""The parity suites again, through the checked build (libpxr_checked.so,
-DPXR_CHECKED): every shared-memory index of the fused render kernel (record,
span, row-owner, queue, fragment and pixel slots, the video texel and
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

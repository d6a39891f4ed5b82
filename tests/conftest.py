import json
import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(REPO, "tests", "golden")
for p in (REPO, os.path.join(REPO, "oracle")):
    if p not in sys.path:
        sys.path.insert(0, p)

MODEL_NAMES = ("cheetah_lite", "walker_lite", "hopper_lite", "ant_lite", "humanoid_lite")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


def pytest_sessionstart(session):
    # tests/test_gpu_checked.py re-runs the GPU suites with PXR_LIB_PATH on
    # the checked build: make sure that is the library that really loads
    if os.environ.get("PXR_EXPECT_CHECKED"):
        from paper_2502_00021_b200 import _native

        assert _native.lib().pxr_build_checked() == 1, _native.LIB_PATH


def pytest_terminal_summary(terminalreporter):
    if os.environ.get("PXR_EXPECT_CHECKED"):
        terminalreporter.write_line("checked build loaded (PXR_DCHECK on)")


def pytest_collection_modifyitems(config, items):
    try:
        import torch

        have_gpu = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        have_gpu = False
    if have_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


def golden(name):
    with np.load(os.path.join(GOLDEN, name), allow_pickle=False) as z:
        return {k: z[k] for k in z.files}


def replay_meta(rec):
    return json.loads(str(rec["meta"]))


def spec_of(name):
    from paper_2502_00021_b200.models import STANDIN_MODELS, builtin_model, load_model

    if name in STANDIN_MODELS:
        return load_model(STANDIN_MODELS[name])
    return builtin_model(name)


def geometry_of(name):
    from paper_2502_00021_b200.models import model_kinematics
    from paper_2502_00021_b200.render import RobotGeometry

    _, _, length, radius = model_kinematics(spec_of(name))
    return RobotGeometry(length, radius)


@pytest.fixture(scope="session")
def oracle():
    import oracle as O

    O.build()
    return O


@pytest.fixture(scope="module")
def torch():
    import torch as _t

    return _t


@pytest.fixture(scope="module")
def pkg():
    """The package with its CUDA library loaded (GPU tests)."""
    import paper_2502_00021_b200 as P

    P._native.lib()
    return P


class _Knobs:
    """PXR_DEBUG_* knobs of the loaded library (pxr_set_debug), unset again
    at teardown."""

    def __init__(self):
        self._set = []

    def set(self, name, value):
        from paper_2502_00021_b200 import _native

        _native.set_debug(name, value)
        self._set.append(name)

    def clear(self):
        from paper_2502_00021_b200 import _native

        for name in reversed(self._set):
            _native.set_debug(name, None)
        self._set.clear()


@pytest.fixture
def knobs():
    k = _Knobs()
    yield k
    k.clear()

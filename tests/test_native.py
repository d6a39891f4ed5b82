"""The C-ABI library builds for sm_100a, loads without a GPU and exports
every entry point include/pxr.h declares; argument validation happens before
any CUDA call (reference convention: ValueError before any kernel runs)."""

import ctypes
import os
import re
import subprocess

import pytest

from conftest import REPO

HEADER = os.path.join(REPO, "include", "pxr.h")


def declared_symbols():
    with open(HEADER) as f:
        src = f.read()
    return sorted(set(re.findall(r"^\s*(?:pxr_status|int32_t|const char \*)\s*(pxr_\w+)\(",
                                 src, re.M)))


@pytest.fixture(scope="module")
def native():
    import paper_2502_00021_b200._native as N

    N.build()
    return N


def test_header_declares_entry_points():
    syms = declared_symbols()
    assert "pxr_render_step" in syms and len(syms) >= 12


def test_library_exports_every_declared_symbol(native):
    lib = native.lib()
    for s in declared_symbols():
        assert hasattr(lib, s), s
    assert set(declared_symbols()) == set(native.EXPORTED)


def test_abi_and_status_strings(native):
    lib = native.lib()
    assert lib.pxr_abi_version() == 3
    assert lib.pxr_status_string(1) == b"invalid argument"
    if native.LIB_PATH.endswith("libpxr.so"):
        assert lib.pxr_build_checked() == 0  # the product build has no device checks


def test_checked_build_exports_the_same_abi(native):
    """libpxr_checked.so (make checked): the same kernels with PXR_DCHECK
    bounds checks, loaded only by tests/test_gpu_checked.py."""
    path = os.path.join(os.path.dirname(native.LIB_PATH), "libpxr_checked.so")
    if not os.path.exists(path):
        subprocess.run(["make", "-s", "-C", native.CSRC, "checked"], check=True)
    chk = ctypes.CDLL(path)
    for s in declared_symbols():
        assert hasattr(chk, s), s
    chk.pxr_build_checked.restype = ctypes.c_int32
    assert chk.pxr_build_checked() == 1


def test_sm100a_cubin_present(native):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", native.LIB_PATH],
                         capture_output=True, text=True, check=True).stdout
    assert "sm_100a" in out


def test_validation_without_gpu(native):
    lib = native.lib()
    g = native.Geometry(None, None, None, None, 0, 0, 4)
    cam = native.Camera()
    d = native.Distractor(native.MODE_NONE)
    st = lib.pxr_render_step(ctypes.byref(g), ctypes.byref(cam), None, 0, 84, 84, 0,
                             ctypes.byref(d), None, 0, None, None, 0, None, None, None)
    assert st == native.PXR_ERR_INVALID
    assert b"batch" in lib.pxr_last_error()
    st = lib.pxr_render_step(ctypes.byref(g), ctypes.byref(cam), 1, 1, 4, 84, 0,
                             ctypes.byref(d), None, 0, None, None, 0, 1, None, None)
    assert st == native.PXR_ERR_INVALID
    with pytest.raises(ValueError):
        native.check(st)
    d = native.Distractor(7)
    st = lib.pxr_render_step(ctypes.byref(g), ctypes.byref(cam), 1, 1, 84, 84, 0,
                             ctypes.byref(d), None, 0, None, None, 0, 1, None, None)
    assert st == native.PXR_ERR_INVALID
    assert lib.pxr_apply_color(None, None, 1, 8, 8, None) == native.PXR_ERR_INVALID
    assert lib.pxr_grayscale(None, None, 4, None) == native.PXR_ERR_INVALID
    # ABI v2: the standalone distractor advance takes host keys only
    d = native.Distractor(native.MODE_COLOR)
    keys = native.StepKeys(1, 2, 0, 4, 12345)
    st = lib.pxr_advance_distractors(ctypes.byref(d), None, 4, ctypes.byref(keys), None, None)
    assert st == native.PXR_ERR_UNSUPPORTED and b"device_key" in lib.pxr_last_error()
    assert lib.pxr_step_key_advance(0, 0, None, None, None) == native.PXR_ERR_INVALID


def test_product_never_imports_oracle():
    pkg = os.path.join(REPO, "paper_2502_00021_b200")
    for root, _, files in os.walk(pkg):
        for fn in files:
            if fn.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                with open(os.path.join(root, fn)) as f:
                    src = f.read()
                assert "import oracle" not in src and "oracle/" not in src.replace(
                    "oracle/,", ""), fn


def test_cpu_has_no_fallback(native, monkeypatch):
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2502_00021_b200 as P

    with pytest.raises(RuntimeError):
        P.render_robot_batch(P.RobotGeometry([0.5], [0.05]), [[[0.0, 0.6, 0.0]]],
                             P.CameraConfig(), 84, 84, False)


def test_debug_knobs_set_and_unset(native):
    """pxr_set_debug: the run-time override of the PXR_DEBUG_* environment
    (read once by the library); unknown names are a ValueError."""
    from paper_2502_00021_b200 import _native

    _native.set_debug("PXR_DEBUG_BAND_H", 12)
    _native.set_debug("PXR_DEBUG_BAND_H", None)
    with pytest.raises(ValueError):
        _native.set_debug("PXR_DEBUG_NOT_A_KNOB", 1)

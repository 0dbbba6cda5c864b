"""C-ABI library: builds for sm_100a, loads, exports every symbol include/mhfd.h
declares, and validates arguments before touching the device (CPU-only tests)."""
import ctypes
import os
import re
import subprocess

import pytest
import torch

from paper_2108_12050_b200 import _abi, _build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "mhfd.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(mhfd_[a-z_0-9]+)\s*\(", src)))


def test_library_builds_and_exports_every_declared_symbol():
    lib = _abi.load()
    declared = _declared()
    assert set(declared) == set(_abi.EXPORTS), declared
    out = subprocess.run(["nm", "-D", "--defined-only", _build.LIB], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (mhfd_[a-z_0-9]+)$", out, flags=re.M))
    missing = [s for s in declared if s not in exported]
    assert not missing, missing
    for s in declared:
        assert hasattr(lib, s)
    assert lib.mhfd_abi_version() == 4


def test_library_is_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", _build.LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out.replace("sm_100a", ""))


def test_status_strings():
    lib = _abi.load()
    for code, name in _abi.STATUS.items():
        assert lib.mhfd_status_string(code).decode() == name


def test_params_default_and_struct_size():
    p = _abi.mhfd_params()
    _abi.load().mhfd_params_default(ctypes.byref(p))
    assert p.struct_size == ctypes.sizeof(_abi.mhfd_params)
    assert (p.min_sigma, p.max_sigma, p.num_scales) == (1.0, 10.0, 10)
    assert p.sat_low == pytest.approx(0.00175) and p.nms == 0 and p.strict == 0 and p.polarity == 0


def test_abi1_struct_size_reads_polarity_as_dark():
    """An ABI-1 caller's struct (without `polarity`) is accepted; validation still runs."""
    lib = _abi.load()
    p = _abi.mhfd_params()
    lib.mhfd_params_default(ctypes.byref(p))
    p.width, p.height, p.max_sigma = 256, 256, 5.0
    p.struct_size = _abi.mhfd_params.polarity.offset   # ABI 1 layout
    p.polarity = 7                                     # beyond struct_size: ignored
    p.min_sigma = 0.0                                  # still validated
    h = ctypes.c_void_p()
    assert lib.mhfd_create(ctypes.byref(p), ctypes.byref(h)) == 1
    assert "min_sigma" in lib.mhfd_last_error().decode()


@pytest.mark.parametrize("field,value,status", [
    ("min_sigma", 0.0, 1), ("max_sigma", 0.5, 1), ("num_scales", 0, 1), ("num_scales", 63, 1),
    ("threshold", -1.0, 1), ("threshold", float("nan"), 1), ("overlap", 1.5, 1), ("sat_low", 0.6, 1),
    ("nms", 7, 1), ("strict", 2, 1), ("max_sigma", 40.0, 1), ("width", 50, 2), ("height", 70000, 2),
    ("polarity", 2, 1), ("struct_size", 8, 1), ("response", 2, 1), ("schedule", 9, 1), ("schedule", -1, 1),
])
def test_create_validates_before_device(field, value, status):
    lib = _abi.load()
    p = _abi.mhfd_params()
    lib.mhfd_params_default(ctypes.byref(p))
    p.width, p.height, p.max_sigma = 256, 256, 5.0
    setattr(p, field, value)
    h = ctypes.c_void_p()
    assert lib.mhfd_create(ctypes.byref(p), ctypes.byref(h)) == status
    assert lib.mhfd_last_error().decode()


def test_create_without_gpu_reports_device():
    lib = _abi.load()
    p = _abi.mhfd_params()
    lib.mhfd_params_default(ctypes.byref(p))
    p.width = p.height = 256
    h = ctypes.c_void_p()
    st = lib.mhfd_create(ctypes.byref(p), ctypes.byref(h))
    if torch.cuda.is_available():
        assert st == 0
        lib.mhfd_destroy(h)
    else:
        assert st == 6 and "device" in lib.mhfd_last_error().decode()


def test_null_and_destroy_safe():
    lib = _abi.load()
    lib.mhfd_destroy(None)
    n = ctypes.c_size_t()
    assert lib.mhfd_workspace_bytes(None, 1, ctypes.byref(n)) == 1
    assert lib.mhfd_focus_score(None, None, 1, 1, 256, None, 0, None, None, None) == 1


@pytest.mark.parametrize("args,status", [
    # (dtype, W, H, in_pitch, factor, out_pitch, batch) -> status; pointers are dummies:
    # validation runs before any device work
    ((1, 16, 16, 16, 0, 16, 1), 1),      # factor 0
    ((1, 16, 8, 16, 9, 16, 1), 1),       # factor > min(W, H)
    ((3, 16, 16, 16, 2, 16, 1), 1),      # bad dtype
    ((1, 16, 16, 16, 2, 16, -1), 1),     # negative batch
    ((1, 16, 16, 8, 2, 8, 1), 2),        # input pitch < row
    ((1, 16, 16, 16, 2, 4, 1), 2),       # output pitch < ceil(W/f)
    ((2, 16, 16, 33, 2, 16, 1), 2),      # u16 pitch not a multiple of 2
    ((1, 0, 16, 16, 1, 16, 1), 2),       # empty width
])
def test_downsample_validates_before_device(args, status):
    lib = _abi.load()
    dt, W, H, ip, f, op, B = args
    dummy = ctypes.c_void_p(0x1000)
    assert lib.mhfd_downsample(dummy, dt, W, H, ip, f, dummy, op, B, None) == status
    assert lib.mhfd_downsample(None, 1, 16, 16, 16, 1, dummy, 16, 1, None) == 1
    # batch 0 is a valid no-op that enqueues nothing
    assert lib.mhfd_downsample(dummy, 1, 16, 16, 16, 2, dummy, 8, 0, None) == 0


@pytest.mark.parametrize("W,n,status", [(300, 10, 2), (256, 32, 1)])
def test_log_response_validates_before_device(W, n, status):
    # the LoG response (reading R23) runs the two-pass kernels: width % 256 == 0 and
    # 2n sub-levels within the level table
    lib = _abi.load()
    p = _abi.mhfd_params()
    lib.mhfd_params_default(ctypes.byref(p))
    p.width, p.height, p.max_sigma, p.num_scales = W, 256, 5.0, n
    p.response = _abi.MHFD_RESPONSE_LOG
    h = ctypes.c_void_p()
    assert lib.mhfd_create(ctypes.byref(p), ctypes.byref(h)) == status
    assert "LoG" in lib.mhfd_last_error().decode()


def test_abi2_struct_size_reads_response_as_dog():
    # an ABI-2 caller's struct ends before `response`: the field beyond struct_size is not
    # read (a garbage value there must not be validated)
    lib = _abi.load()
    p = _abi.mhfd_params()
    lib.mhfd_params_default(ctypes.byref(p))
    p.width, p.height, p.max_sigma = 256, 256, 5.0
    p.struct_size = _abi.mhfd_params.response.offset
    p.response = 9
    p.min_sigma = 0.0
    h = ctypes.c_void_p()
    assert lib.mhfd_create(ctypes.byref(p), ctypes.byref(h)) == 1
    assert "min_sigma" in lib.mhfd_last_error().decode()


@pytest.mark.parametrize("W,b,status", [(300, 1, 2), (256, 2, 1)])
def test_boundary_validates_before_device(W, b, status):
    # reflect (reading R25) runs the two-pass kernels: width % 256 == 0; unknown values rejected
    lib = _abi.load()
    p = _abi.mhfd_params()
    lib.mhfd_params_default(ctypes.byref(p))
    p.width, p.height, p.max_sigma = W, 256, 5.0
    p.boundary = b
    h = ctypes.c_void_p()
    assert lib.mhfd_create(ctypes.byref(p), ctypes.byref(h)) == status
    assert "boundary" in lib.mhfd_last_error().decode()


def test_abi3_struct_size_reads_schedule_as_auto():
    # an ABI-3 caller's struct ends before `schedule` (ABI 4): a garbage value there is not read
    lib = _abi.load()
    p = _abi.mhfd_params()
    lib.mhfd_params_default(ctypes.byref(p))
    assert p.schedule == 0
    p.width, p.height, p.max_sigma = 256, 256, 5.0
    p.struct_size = _abi.mhfd_params.schedule.offset
    p.schedule = 9
    p.min_sigma = 0.0
    h = ctypes.c_void_p()
    assert lib.mhfd_create(ctypes.byref(p), ctypes.byref(h)) == 1
    assert "min_sigma" in lib.mhfd_last_error().decode()

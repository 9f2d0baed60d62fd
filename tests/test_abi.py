"""The C-ABI library builds for sm_100a, loads without a GPU and exports every
symbol include/slim.h declares (no compute calls: -m "not gpu")."""
import ctypes
import os
import re
import subprocess

import pytest

import paper_2510_09018_b200 as slim
from paper_2510_09018_b200 import build as slim_build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    hdr = open(os.path.join(ROOT, "include", "slim.h")).read()
    return sorted(set(re.findall(r"SLIM_API[^;(]*?\b(slim_\w+)\s*\(", hdr)))


def test_header_declares_the_north_star_calls():
    names = _declared()
    for n in ("slim_load_segment", "slim_forward", "slim_forward_chain", "slim_pack", "slim_launch"):
        assert n in names


def test_library_exports_every_declared_symbol():
    slim_build.build()
    lib = ctypes.CDLL(slim.LIB_PATH)
    missing = [n for n in _declared() if not hasattr(lib, n)]
    assert not missing, missing
    assert sorted(slim.EXPORTED) == _declared()


def test_exports_are_exactly_the_abi():
    out = subprocess.check_output(["nm", "-D", "--defined-only", slim.LIB_PATH], text=True)
    exported = sorted({l.split()[-1] for l in out.splitlines() if l.split()[-2] == "T" and l.split()[-1].startswith("slim_")})
    assert exported == _declared()


def test_sass_contains_tcgen05_and_tma():
    """The conv kernel is tcgen05 + TMA code (UTCHMMA / UTMALDG / UTMASTG / LDTM in SASS)."""
    sass = subprocess.check_output(["/usr/local/cuda/bin/cuobjdump", "-sass", slim.LIB_PATH], text=True)
    for mnem in ("UTCHMMA", "UTMALDG", "UTMASTG", "LDTM"):
        assert mnem in sass, mnem
    assert "HMMA" not in re.sub(r"UTCHMMA", "", sass)   # no legacy mma.sync path


def test_status_strings_and_channels():
    lib = slim.load_library()
    assert lib.slim_status_str(-1) == b"SLIM_EINVAL"
    assert [slim.slim_channels(r, 64) for r in (0.25, 0.5, 0.75, 1.0)] == [16, 32, 48, 64]
    assert slim.slim_channels(0.75, 512) == 384


def test_create_without_gpu_fails_loudly():
    """No CPU fallback: creating a context without a usable GPU is an error, not a silent path."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(slim.SlimError):
        slim.slim_create(0, slim.default_config())


def test_segment_bytes_scales_like_w_squared():
    """CANLOAD's byte estimate: conv weights scale with r_prev*r or r^2 (SPEC param_bytes = P_s w^2)."""
    cfg = slim.default_config()
    b1 = slim.slim_segment_bytes(cfg, 2, 1.0, 1.0)
    b5 = slim.slim_segment_bytes(cfg, 2, 0.5, 0.5)
    assert 0.24 < b5 / b1 < 0.26
    assert slim.slim_segment_bytes(cfg, 2, 0.3, 0.5) == 0          # width outside the set


def test_groupnorm_config_validation():
    """GN groups must tile every active width (reading R16): rejected before any device call."""
    lib = slim.load_library()
    h = ctypes.c_void_p()
    for g in (24, 4, 12):
        cfg = slim.default_config(norm="gn", gn_group_channels=g)
        assert lib.slim_create(0, ctypes.byref(cfg), ctypes.byref(h)) == slim.SLIM_EUNSUPPORTED
    cfg = slim.default_config(norm=7)
    assert lib.slim_create(0, ctypes.byref(cfg), ctypes.byref(h)) == slim.SLIM_EINVAL
    cfg = slim.default_config()
    assert cfg.norm == slim.SLIM_NORM_BN and cfg.gn_group_channels == 16


def test_stream_executor_rejects_bad_arguments_without_gpu():
    """slim_stream_*: argument checks come before any CUDA call (NULL context / handle)."""
    lib = slim.load_library()
    h = ctypes.c_void_p(1)
    assert lib.slim_stream_create(None, 16, 8, 1, ctypes.byref(h)) == -1 and h.value is None
    assert lib.slim_stream_create(None, 16, 8, 1, None) == -1
    assert lib.slim_stream_run(None, None, None, 4, None, None, None) == -1
    lib.slim_stream_destroy(None)

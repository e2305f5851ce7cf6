"""CPU: the C-ABI library loads and exports every symbol include/mshbm.h
declares; host-only entry points (schedules, config validation) agree with
the reference semantics.  No GPU compute is called here."""

import ctypes as C
import os
import re
import subprocess

import pytest

from mshbm_testutil import ROOT

HEADER = os.path.join(ROOT, "include", "mshbm.h")


@pytest.fixture(scope="module")
def lib():
    from paper_1901_09593_b200.build import build
    build()
    from paper_1901_09593_b200 import _lib
    return _lib.load_library()


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(mshbm_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_entry_points():
    names = declared_functions()
    assert "mshbm_run_pipeline" in names and "mshbm_engine_at" in names
    assert len(names) >= 20


def test_library_exports_every_declared_symbol(lib):
    from paper_1901_09593_b200 import _lib
    for name in declared_functions():
        assert hasattr(lib, name), name
        assert name in _lib.SIGNATURES, f"{name} not bound in _lib.SIGNATURES"
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH],
                         capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (mshbm_\w+)", out))
    assert set(declared_functions()) <= exported


def test_library_is_sm100a(lib):
    from paper_1901_09593_b200 import _lib
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_schedules_match_reference_literals(lib):
    # pkg/tests/test_pyramid.py:44-51
    assert [lib.mshbm_level_d_max(64, k) for k in range(3)] == [64, 32, 16]
    assert [lib.mshbm_level_block(11, k) for k in range(3)] == [11, 5, 3]
    assert lib.mshbm_level_d_max(5, 4) == 1
    assert lib.mshbm_level_block(9, 1) == 3
    assert lib.mshbm_level_block(7, 5) == 3
    out = C.c_int32()
    assert lib.mshbm_auto_levels(2960, 2016, 256, 11, C.byref(out)) == 0
    assert out.value == 5                      # pkg/tests/test_pyramid.py:96-98


@pytest.mark.parametrize("kw,code", [
    (dict(d_max=0), 2), (dict(alpha=0.0), 2), (dict(alpha=1.01), 2), (dict(beta=1.0), 2),
    (dict(block=4), 2), (dict(block=1), 2), (dict(sigma_eps=0.0), 2), (dict(sign=7), 2),
])
def test_config_validation_codes(lib, kw, code):
    from paper_1901_09593_b200 import _lib
    base = dict(d_max=16, levels=-1, block=5, radius=1, alpha=0.9, beta=0.9,
                sigma_eps=1e-6, sign=0)
    base.update(kw)
    cfg = _lib.Config(**base)
    out = C.c_int32()
    assert lib.mshbm_resolve_levels(C.byref(cfg), 64, 64, C.byref(out)) == code


def test_resolve_levels_depth_errors(lib):
    from paper_1901_09593_b200 import _lib
    cfg = _lib.Config(d_max=64, levels=6, block=5, radius=1, alpha=0.9, beta=0.9,
                      sigma_eps=1e-6, sign=0)
    out = C.c_int32()
    assert lib.mshbm_resolve_levels(C.byref(cfg), 64, 64, C.byref(out)) == 1   # too deep
    cfg.levels = 2
    assert lib.mshbm_resolve_levels(C.byref(cfg), 375, 450, C.byref(out)) == 0
    assert out.value == 2


def test_python_config_mirror():
    from paper_1901_09593_b200 import ConfigError, MatchConfig
    for kw in [dict(d_max=0), dict(d_max=16, alpha=0.0), dict(d_max=16, beta=1.0),
               dict(d_max=16, block=4), dict(d_max=16, levels=-1),
               dict(d_max=16, sigma_eps=0.0), dict(d_max=16, sign="up"),
               dict(d_max=16, radius=-1)]:
        with pytest.raises(ConfigError):
            MatchConfig(**kw)
    assert MatchConfig(d_max=8).radius == 1

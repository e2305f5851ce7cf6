"""CPU: the native codecs (csrc/codec.cu) against the reference's own
formats.py -- decoded arrays, byte-identical writer output, and the same
exception class and message for every malformed input
(tests/golden/formats.npz, tools/make_golden.py formats_cases)."""

import os

import numpy as np
import pytest

from mshbm_testutil import GOLDEN

F = pytest.importorskip("paper_1901_09593_b200.formats")


@pytest.fixture(scope="module")
def g():
    return np.load(os.path.join(GOLDEN, "formats.npz"))


def _write(tmp_path, name, arr):
    p = tmp_path / name
    p.write_bytes(bytes(arr))
    return p


@pytest.mark.parametrize("name", ["p5", "p2", "p6_16", "p3", "p6_8", "pgm8", "pgm_preview",
                                  "pgm16", "pgm_half"])
def test_read_pnm_matches_reference(g, tmp_path, name):
    got = F.read_pnm(_write(tmp_path, name, g[f"file_{name}"]))
    np.testing.assert_allclose(got, g[f"dec_{name}"], rtol=0, atol=1e-15)


@pytest.mark.parametrize("name", ["pfm_le", "pfm_be", "pfm_s2"])
def test_read_pfm_matches_reference(g, tmp_path, name):
    got = F.read_pfm(_write(tmp_path, name, g[f"file_{name}"]))
    np.testing.assert_array_equal(got.invalid, g[f"inv_{name}"])
    np.testing.assert_array_equal(got.values, g[f"dec_{name}"])   # NaN == NaN here


@pytest.mark.parametrize("name,kw", [("pfm_le", dict(scale=-1.0)), ("pfm_be", dict(scale=1.0)),
                                     ("pfm_s2", dict(scale=-2.5))])
def test_write_pfm_bytes_identical(g, tmp_path, name, kw):
    p = tmp_path / "o.pfm"
    F.write_pfm(g["src_v"], p, **kw)
    assert p.read_bytes() == bytes(g[f"file_{name}"])


def test_write_pgm_bytes_identical(g, tmp_path):
    cases = {"pgm8": (g["src_v"], {}), "pgm_preview": (g["src_dsp"], dict(scale_max=70.0)),
             "pgm16": (g["src_v"], dict(maxval=4095)),
             "pgm_half": (np.array([[0.5 / 255, 1.5 / 255, 2.5 / 255, 253.5 / 255]]), {})}
    for name, (v, kw) in cases.items():
        p = tmp_path / f"{name}.pgm"
        F.write_pgm(v, p, **kw)
        assert p.read_bytes() == bytes(g[f"file_{name}"]), name


def test_malformed_inputs_raise_reference_classes(g, tmp_path):
    for k, (kind, msg) in enumerate(zip(g["bad_kind"], g["bad_msg"])):
        data = bytes(g[f"bad_{k}"])
        p = _write(tmp_path, f"bad{k}", g[f"bad_{k}"])
        reader = F.read_pfm if data[:1] == b"P" and data[1:2] in (b"f", b"F") else F.read_pnm
        with pytest.raises(getattr(F, str(kind))) as ei:
            reader(p)
        assert type(ei.value).__name__ == str(kind)
        assert str(ei.value) == str(msg), (k, str(ei.value), str(msg))


def test_write_errors(tmp_path):
    with pytest.raises(ValueError):
        F.write_pgm(np.zeros((0, 4)), tmp_path / "e.pgm")
    with pytest.raises(ValueError):
        F.write_pfm(np.zeros((0, 4)), tmp_path / "e.pfm")
    with pytest.raises(ValueError):
        F.write_pfm(np.zeros((2, 2)), tmp_path / "e.pfm", scale=0.0)
    with pytest.raises(ValueError):
        F.write_pgm(np.zeros((2, 2)), tmp_path / "e.pgm", maxval=0)
    with pytest.raises(ValueError):
        F.write_pgm(np.zeros((2, 2)), tmp_path / "e.pgm", scale_max=0.0)


def test_exception_hierarchy():
    for cls in (F.MalformedHeaderError, F.TruncatedPayloadError, F.UnsupportedMaxvalError,
                F.MissingKeyError):
        assert issubclass(cls, F.DecodeError) and issubclass(cls, ValueError)


def test_calib(tmp_path):
    p = tmp_path / "calib.txt"
    p.write_text("cam0=[100 0 50]\nndisp=70\n")
    assert F.read_calib(p).ndisp == 70
    p.write_text("ndisp=290\nwidth=2960\nheight=2016\n")
    c = F.read_calib(p)
    assert (c.ndisp, c.width, c.height) == (290, 2960, 2016)
    p.write_text("width=100\nheight=100\n")
    with pytest.raises(F.MissingKeyError):
        F.read_calib(p)
    p.write_text("ndisp=0\n")
    with pytest.raises(F.MalformedHeaderError):
        F.read_calib(p)
    p.write_text("ndisp=abc\n")
    with pytest.raises(F.MalformedHeaderError):
        F.read_calib(p)

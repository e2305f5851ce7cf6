"""Wire formats either side of the disparity path,
mirroring ``/root/reference/pkg/src/pyrstereo/formats.py``.

The codecs are native (``csrc/codec.cu`` in libmshbm, C ABI in
``include/mshbm.h``); this module keeps the reference's names, arguments,
return types and exception classes:

* ``read_pnm`` (P2/P3/P5/P6, maxval <= 65535, BT.601 luma for colour) ->
  (H, W) float64 in [0, 1]                         (formats.py:123-190)
* ``read_pfm`` -> ``GroundTruthDisparity`` (+inf/NaN -> invalid)  (193-232)
* ``write_pfm`` / ``write_pgm``                                  (235-278)
* ``read_calib`` -> ``CalibInfo``                                 (281-312)

Plus the device path the reference has no counterpart for:
``load_pnm_device`` uploads the raw binary samples (1-2 bytes per channel)
and decodes them to an fp32 CUDA tensor, the input ``run_pipeline_device``
takes; ``write_disparity_pfm`` encodes a device or host map.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from .scoring import GroundTruthDisparity

__all__ = ["DecodeError", "MalformedHeaderError", "TruncatedPayloadError",
           "UnsupportedMaxvalError", "MissingKeyError", "GroundTruthDisparity", "CalibInfo",
           "read_pnm", "read_pfm", "write_pfm", "write_pgm", "read_calib", "load_pnm_device",
           "write_disparity_pfm"]


class DecodeError(ValueError):
    """A file could not be decoded."""


class MalformedHeaderError(DecodeError):
    """Magic number, dimensions or scale line are unusable."""


class TruncatedPayloadError(DecodeError):
    """The pixel payload ends before width*height samples."""


class UnsupportedMaxvalError(DecodeError):
    """PNM maxval outside [1, 65535]."""


class MissingKeyError(DecodeError):
    """A required key is absent from a calibration file."""


_EXC = {
    _lib.MSHBM_ERR_DECODE: DecodeError,
    _lib.MSHBM_ERR_MALFORMED: MalformedHeaderError,
    _lib.MSHBM_ERR_TRUNCATED: TruncatedPayloadError,
    _lib.MSHBM_ERR_MAXVAL: UnsupportedMaxvalError,
    _lib.MSHBM_ERR_MISSING_KEY: MissingKeyError,
}


@dataclass(frozen=True)
class CalibInfo:
    """ndisp (required) and optional image dimensions of a calib.txt."""

    ndisp: int
    width: int | None = None
    height: int | None = None


def _raise(status: int) -> None:
    if status == _lib.MSHBM_OK:
        return
    msg = _lib.lib().mshbm_last_error(None)
    msg = msg.decode() if msg else _lib.lib().mshbm_status_string(status).decode()
    exc = _EXC.get(status)
    if exc is not None:
        raise exc(msg)
    if status == _lib.MSHBM_ERR_VALUE:
        raise ValueError(msg)
    raise _lib.MshbmError(f"libmshbm: {msg}")


def _read(path) -> bytes:
    with open(path, "rb") as fh:
        return fh.read()


def _pnm_header(buf: bytes):
    hdr = _lib.PnmHeader()
    _raise(_lib.lib().mshbm_pnm_parse(buf, len(buf), C.byref(hdr)))
    return hdr


def read_pnm(path) -> np.ndarray:
    """PGM/PPM file -> grayscale (H, W) float64 in [0, 1]."""
    buf = _read(path)
    hdr = _pnm_header(buf)
    out = np.empty((hdr.height, hdr.width), dtype=np.float64)
    _raise(_lib.lib().mshbm_pnm_decode(buf, len(buf), C.byref(hdr),
                                       out.ctypes.data_as(C.c_void_p), hdr.width))
    return out


def read_pfm(path) -> GroundTruthDisparity:
    """Single-channel PFM -> values (NaN at non-finite samples) + invalid mask."""
    buf = _read(path)
    hdr = _lib.PfmHeader()
    _raise(_lib.lib().mshbm_pfm_parse(buf, len(buf), C.byref(hdr)))
    values = np.empty((hdr.height, hdr.width), dtype=np.float64)
    invalid = np.empty((hdr.height, hdr.width), dtype=np.uint8)
    _raise(_lib.lib().mshbm_pfm_decode(buf, len(buf), C.byref(hdr),
                                       values.ctypes.data_as(C.c_void_p),
                                       invalid.ctypes.data_as(C.c_void_p), hdr.width))
    return GroundTruthDisparity(values=values, invalid=invalid.astype(bool))


def _encode(fn, values, *args) -> bytes:
    v = np.ascontiguousarray(np.asarray(values, dtype=np.float64))
    if v.ndim != 2 or v.size == 0:
        raise ValueError(f"expected a non-empty 2-D array, got shape {v.shape}")
    h, w = v.shape
    size = fn(v.ctypes.data_as(C.c_void_p), h, w, w, *args, None, 0)
    if size < 0:
        _raise(-size)
    out = (C.c_uint8 * size)()
    fn(v.ctypes.data_as(C.c_void_p), h, w, w, *args, out, size)
    return bytes(out)


def write_pfm(values, path, scale: float = -1.0) -> None:
    """2-D array -> grayscale PFM (NaN stored as +inf; scale sign = byte order)."""
    if scale == 0.0:
        raise ValueError("scale must be nonzero")
    data = _encode(_lib.lib().mshbm_pfm_encode, values, float(scale))
    with open(path, "wb") as fh:
        fh.write(data)


def write_pgm(values, path, maxval: int = 255, scale_max: float = 1.0) -> None:
    """2-D array -> binary PGM, [0, scale_max] mapped onto [0, maxval]."""
    if not 1 <= maxval <= 65535:
        raise ValueError(f"maxval {maxval} outside [1, 65535]")
    if scale_max <= 0:
        raise ValueError("scale_max must be positive")
    data = _encode(_lib.lib().mshbm_pgm_encode, values, int(maxval), float(scale_max))
    with open(path, "wb") as fh:
        fh.write(data)


def read_calib(path) -> CalibInfo:
    """Middlebury calib.txt: ndisp (required), width/height (optional)."""
    entries: dict[str, str] = {}
    with open(path, "r", encoding="ascii", errors="replace") as fh:
        for line in fh:
            line = line.strip()
            if not line or "=" not in line:
                continue
            key, _, value = line.partition("=")
            entries[key.strip()] = value.strip()

    def number(key: str) -> int:
        try:
            return int(float(entries[key]))
        except ValueError:
            raise MalformedHeaderError(f"bad {key} value {entries[key]!r}") from None

    if "ndisp" not in entries:
        raise MissingKeyError("calib file lacks an ndisp entry")
    ndisp = number("ndisp")
    if ndisp < 1:
        raise MalformedHeaderError(f"ndisp must be >= 1, got {ndisp}")
    return CalibInfo(ndisp=ndisp,
                     width=number("width") if "width" in entries else None,
                     height=number("height") if "height" in entries else None)


def load_pnm_device(path, device=None):
    """Binary PGM/PPM -> (H, W) float32 CUDA tensor in [0, 1].  The raw
    samples cross PCIe; decoding (and the range check) runs on the GPU.
    ASCII files are decoded on the host and uploaded as fp32."""
    import torch
    buf = _read(path)
    hdr = _pnm_header(buf)
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
    if hdr.ascii:
        return torch.from_numpy(read_pnm(path).astype(np.float32)).to(dev)
    _lib.context(dev.index)
    host = torch.frombuffer(bytearray(buf), dtype=torch.uint8).pin_memory()
    out = torch.empty((hdr.height, hdr.width), dtype=torch.float32, device=dev)
    with torch.cuda.device(dev):
        _raise(_lib.lib().mshbm_pnm_upload(C.c_void_p(host.data_ptr()), len(buf), C.byref(hdr),
                                           C.c_void_p(out.data_ptr()), hdr.width,
                                           _lib.current_stream()))
    return out


def write_disparity_pfm(disparity, path, scale: float = -1.0) -> None:
    """Disparity map (numpy, or CUDA tensor of int16/float) -> PFM."""
    try:
        import torch
        if isinstance(disparity, torch.Tensor):
            disparity = disparity.detach().to("cpu").double().numpy()
    except ImportError:   # pragma: no cover
        pass
    write_pfm(np.asarray(disparity, dtype=np.float64), path, scale)

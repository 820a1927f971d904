"""NIfTI-1 single-file volumes and raw + JSON warp fields (nifti.hpp:24-303): the data
formats either side of the registration path, byte-compatible with the reference.

Volumes are numpy arrays (nz, ny, nx) (x fastest, volume.hpp:41-43) or CUDA tensors;
readers return fp64 values like the reference (``NiftiVolume.volume``) and
``to_device`` uploads them as the fp32 volumes the kernels take. Errors raise
``FormatError`` (with the byte offset) and ``IoError`` like the reference.
"""
from __future__ import annotations

import json
import struct
from dataclasses import dataclass, field
from typing import Tuple

import numpy as np

HEADER_BYTES = 348  # kNiftiHeaderBytes (nifti.hpp:54)
VOX_OFFSET = 352    # kNiftiVoxOffset (nifti.hpp:55)
_DTYPES = {2: np.uint8, 4: np.int16, 16: np.float32, 64: np.float64}


class FormatError(RuntimeError):
    """FormatError (nifti.hpp:24-28): a malformed file, with the offending byte offset."""

    def __init__(self, what: str, offset: int):
        super().__init__(f"{what} (at byte {offset})")
        self.offset = offset


class IoError(RuntimeError):
    """IoError (nifti.hpp:30-32)."""


@dataclass
class NiftiHeader:
    """NiftiHeader (nifti.hpp:34-45)."""
    dim: Tuple[int, ...] = (0,) * 8
    datatype: int = 0
    bitpix: int = 0
    pixdim: Tuple[float, ...] = (0.0,) * 8
    vox_offset: float = 352.0
    scl_slope: float = 0.0
    scl_inter: float = 0.0
    qoffset: Tuple[float, ...] = (0.0, 0.0, 0.0)
    magic: bytes = b"\0\0\0\0"
    big_endian: bool = False


@dataclass
class NiftiVolume:
    """NiftiVolume (nifti.hpp:47-50): the header and the fp64 volume with its geometry."""
    header: NiftiHeader
    volume: np.ndarray                      # (nz, ny, nx) float64
    spacing: Tuple[float, float, float] = (1.0, 1.0, 1.0)
    origin: Tuple[float, float, float] = (0.0, 0.0, 0.0)

    def to_device(self, device="cuda"):
        import torch
        return torch.from_numpy(np.ascontiguousarray(self.volume, dtype=np.float32)).to(device)


def read_nifti_bytes(b: bytes) -> NiftiVolume:
    """read_nifti_bytes (nifti.hpp:99-176)."""
    if len(b) < HEADER_BYTES:
        raise FormatError("file shorter than header", len(b))
    swap = False
    if struct.unpack_from("<i", b, 0)[0] != 348:
        if struct.unpack_from(">i", b, 0)[0] == 348:
            swap = True
        else:
            raise FormatError("sizeof_hdr is not 348 in either byte order", 0)
    e = ">" if swap else "<"
    h = NiftiHeader(big_endian=swap)
    h.dim = struct.unpack_from(e + "8h", b, 40)
    h.datatype, h.bitpix = struct.unpack_from(e + "2h", b, 70)
    h.pixdim = struct.unpack_from(e + "8f", b, 76)
    h.vox_offset, h.scl_slope, h.scl_inter = struct.unpack_from(e + "3f", b, 108)
    h.qoffset = struct.unpack_from(e + "3f", b, 268)
    h.magic = bytes(b[344:348])
    if h.magic == b"ni1\0":
        raise FormatError('two-file NIfTI (magic "ni1") is unsupported', 344)
    if h.magic != b"n+1\0":
        raise FormatError("bad magic", 344)
    if h.dim[0] < 1 or h.dim[0] > 3:
        raise FormatError("only 3-D volumes supported", 40)
    nx, ny, nz = h.dim[1], (h.dim[2] if h.dim[0] >= 2 else 1), (h.dim[3] if h.dim[0] >= 3 else 1)
    if nx <= 0 or ny <= 0 or nz <= 0:
        raise FormatError("non-positive dims", 40)
    if h.datatype not in _DTYPES:
        raise FormatError(f"unsupported datatype {h.datatype}", 70)
    dt = np.dtype(_DTYPES[h.datatype]).newbyteorder(">" if swap else "<")
    off = int(h.vox_offset)
    n = nx * ny * nz
    if len(b) < off + n * dt.itemsize:
        raise FormatError("truncated payload", len(b))
    v = np.frombuffer(b, dtype=dt, count=n, offset=off).astype(np.float64)
    if h.scl_slope != 0.0:
        v = float(np.float32(h.scl_slope)) * v + float(np.float32(h.scl_inter))
    spacing = tuple(float(s) if s > 0 else 1.0 for s in h.pixdim[1:4])
    origin = tuple(float(q) for q in h.qoffset)
    return NiftiVolume(h, v.reshape(nz, ny, nx), spacing, origin)


def read_nifti(path: str) -> NiftiVolume:
    """read_nifti (nifti.hpp:178-184)."""
    try:
        with open(path, "rb") as fh:
            data = fh.read()
    except OSError:
        raise IoError(f"cannot open {path}") from None
    return read_nifti_bytes(data)


def _header_bytes(shape, spacing, origin, datatype: int, bitpix: int) -> bytearray:
    """nifti_bytes_common (nifti.hpp:188-217): the reference's little-endian header."""
    nz, ny, nx = shape
    if max(nx, ny, nz) > 32767:
        raise ValueError("write_nifti: dims exceed int16 header fields")
    b = bytearray(VOX_OFFSET)
    struct.pack_into("<i", b, 0, 348)
    struct.pack_into("<8h", b, 40, 3, nx, ny, nz, 1, 1, 1, 1)
    struct.pack_into("<2h", b, 70, datatype, bitpix)
    struct.pack_into("<4f", b, 76, 1.0, *[float(s) for s in spacing])
    struct.pack_into("<3f", b, 108, float(VOX_OFFSET), 0.0, 0.0)
    struct.pack_into("<3f", b, 268, *[float(o) for o in origin])
    b[344:348] = b"n+1\0"
    return b


def _host(v) -> np.ndarray:
    if hasattr(v, "detach"):
        v = v.detach().cpu().numpy()
    return np.asarray(v)


def nifti_bytes(v, spacing=(1.0, 1.0, 1.0), origin=(0.0, 0.0, 0.0)) -> bytes:
    """The bytes write_nifti (nifti.hpp:230-239) produces for an fp32 (datatype 16) or
    fp64 (datatype 64) volume."""
    a = _host(v)
    if a.ndim != 3:
        raise ValueError("write_nifti: a (nz, ny, nx) volume is required")
    f64 = a.dtype == np.float64
    b = _header_bytes(a.shape, spacing, origin, 64 if f64 else 16, 64 if f64 else 32)
    return bytes(b) + np.ascontiguousarray(a, dtype="<f8" if f64 else "<f4").tobytes()


def _dump(path: str, data: bytes):
    if not path:
        raise IoError("empty output path")
    try:
        with open(path, "wb") as fh:
            fh.write(data)
    except OSError:
        raise IoError(f"cannot open {path} for writing") from None


def write_nifti(v, path: str, spacing=(1.0, 1.0, 1.0), origin=(0.0, 0.0, 0.0)):
    """write_nifti (nifti.hpp:230-239); a CUDA tensor is read back first."""
    _dump(path, nifti_bytes(v, spacing, origin))


def write_labels(v, path: str, spacing=(1.0, 1.0, 1.0)):
    """write_nifti of a LabelVolume (nifti.hpp:241-251): int16 payload, origin 0."""
    a = _host(v)
    b = _header_bytes(a.shape, spacing, (0.0, 0.0, 0.0), 4, 16)
    _dump(path, bytes(b) + np.ascontiguousarray(a.astype(np.uint16).astype("<i2")).tobytes())


def nifti_to_labels(nv: NiftiVolume) -> np.ndarray:
    """nifti_to_labels (nifti.hpp:253-266): integer labels in [0, 65535]."""
    v = nv.volume.ravel()
    r = np.rint(v)
    bad = np.nonzero((np.abs(v - r) > 1e-6) | (r < 0) | (r > 65535))[0]
    if bad.size:
        raise FormatError("label volume has non-integer values", int(bad[0]))
    return r.astype(np.uint16).reshape(nv.volume.shape)


def write_warp(w, prefix: str, spacing=(1.0, 1.0, 1.0), origin=(0.0, 0.0, 0.0)):
    """write_warp (nifti.hpp:268-286): fp64 raw payload (xyz interleaved) + JSON sidecar."""
    a = _host(w)
    if a.ndim != 4 or a.shape[3] != 3:
        raise ValueError("write_warp: a (nz, ny, nx, 3) field is required")
    _dump(prefix + ".raw", np.ascontiguousarray(a, dtype="<f8").tobytes())
    nz, ny, nx = a.shape[:3]
    meta = {"dims": [nx, ny, nz], "spacing": [float(s) for s in spacing], "origin": [float(o) for o in origin],
            "channels": 3}
    try:
        with open(prefix + ".json", "w") as fh:
            fh.write(json.dumps(meta, indent=2) + "\n")
    except OSError:
        raise IoError(f"cannot open {prefix}.json for writing") from None


def read_warp(prefix: str) -> np.ndarray:
    """read_warp (nifti.hpp:288-303): (nz, ny, nx, 3) float64."""
    try:
        with open(prefix + ".json") as fh:
            meta = json.load(fh)
    except OSError:
        raise IoError(f"cannot open {prefix}.json") from None
    nx, ny, nz = (int(v) for v in meta["dims"])
    if int(meta["channels"]) != 3:
        raise IoError("warp sidecar: channels must be 3")
    try:
        with open(prefix + ".raw", "rb") as fh:
            raw = fh.read()
    except OSError:
        raise IoError(f"cannot open {prefix}.raw") from None
    n = nx * ny * nz * 3
    if len(raw) < 8 * n:
        raise IoError("warp raw payload truncated")
    return np.frombuffer(raw, dtype="<f8", count=n).reshape(nz, ny, nx, 3).copy()

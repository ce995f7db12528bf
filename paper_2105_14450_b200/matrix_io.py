"""The reference's binary matrix files and parameter checkpoints.

CUBE3D matrix file (cube3d/matrix_io.hpp:18-127): magic "CUBE3D\\0", u8 version = 1, u8
dtype (0 = f64, 1 = f32), u64 rows, u64 cols, little-endian, then rows * cols scalars
row-major; round trips are bit-exact. save_layer_params / load_layer_params
(cube3d/transformer.hpp:259-293): one file per global parameter under `prefix`
(`prefix.ln1_gamma.bin`, ...; vectors as 1 x N matrices); partitioning happens on load.
Errors are C3DError("IoError") like the reference's IoError.
"""
from __future__ import annotations

import struct
from typing import Optional

import numpy as np

from ._lib import C3DError

MAGIC = b"CUBE3D\x00"
VERSION = 1
FIELDS = ["ln1_gamma", "ln1_beta", "w_qkv", "b_qkv", "w_out", "b_out", "ln2_gamma", "ln2_beta",
          "w_fc1", "b_fc1", "w_fc2", "b_fc2"]
_IO = 14  # C3D_ERR_IO


def _io(msg: str) -> C3DError:
    return C3DError(_IO, f"IoError: {msg}")


def write_matrix(path: str, m: np.ndarray, dtype: Optional[str] = None) -> None:
    """write_matrix_file: `m` 2-D (or 1-D, written as 1 x N); dtype 'f64' / 'f32'
    (default: f32 for float32 arrays, else f64)."""
    m = np.asarray(m)
    if m.ndim == 1:
        m = m.reshape(1, -1)
    if m.ndim != 2:
        raise _io("matrices are 2-D")
    kind = dtype or ("f32" if m.dtype == np.float32 else "f64")
    code, npdt = (1, "<f4") if kind == "f32" else (0, "<f8")
    try:
        with open(path, "wb") as f:
            f.write(MAGIC + bytes([VERSION, code]) + struct.pack("<QQ", m.shape[0], m.shape[1]))
            f.write(np.ascontiguousarray(m, dtype=npdt).tobytes())
    except OSError as e:
        raise _io(f"cannot open {path} for writing ({e.strerror})") from None


def matrix_file_dtype(path: str) -> int:
    """Peeks the dtype byte (0 f64, 1 f32), like matrix_file_dtype (matrix_io.hpp:112-124)."""
    try:
        with open(path, "rb") as f:
            head = f.read(9)
    except OSError:
        raise _io(f"cannot open {path}") from None
    if len(head) < 7 or head[:7] != MAGIC:
        raise _io(f"bad matrix file magic in {path}")
    if len(head) < 9:
        raise _io(f"truncated matrix file {path}")
    return head[8]


def read_matrix(path: str, dtype: Optional[str] = None) -> np.ndarray:
    """read_matrix_file: returns float64 or float32 per the file; `dtype` ('f64' / 'f32')
    must match the file when given (the reference's typed read)."""
    try:
        with open(path, "rb") as f:
            raw = f.read()
    except OSError:
        raise _io(f"cannot open {path}") from None
    if len(raw) < 7 or raw[:7] != MAGIC:
        raise _io("bad matrix file magic")
    if len(raw) < 9:
        raise _io("truncated matrix file")
    if raw[7] != VERSION:
        raise _io(f"unsupported matrix file version {raw[7]}")
    code = raw[8]
    if code not in (0, 1):
        raise _io(f"matrix file dtype {code} does not match requested scalar")
    if dtype is not None and code != (1 if dtype == "f32" else 0):
        raise _io(f"matrix file dtype {code} does not match requested scalar")
    if len(raw) < 25:
        raise _io("truncated matrix file")
    rows, cols = struct.unpack("<QQ", raw[9:25])
    es = 4 if code == 1 else 8
    body = raw[25:]
    if len(body) < rows * cols * es:
        raise _io("truncated matrix file")
    a = np.frombuffer(body[:rows * cols * es], dtype="<f4" if code == 1 else "<f8")
    return a.reshape(rows, cols).astype(np.float32 if code == 1 else np.float64)


def save_layer_params(gp, prefix: str, dtype: str = "f64") -> None:
    """save_layer_params (transformer.hpp:259-275) of a GlobalLayerParams."""
    for f in FIELDS:
        write_matrix(f"{prefix}.{f}.bin", np.asarray(getattr(gp, f)), dtype)


def load_layer_params(prefix: str):
    """load_layer_params (transformer.hpp:277-293) -> GlobalLayerParams (float64)."""
    from .cube3d import GlobalLayerParams
    vals = {}
    for f in FIELDS:
        m = read_matrix(f"{prefix}.{f}.bin").astype(np.float64)
        vals[f] = m.reshape(-1) if f.startswith(("ln", "b_")) else m
    return GlobalLayerParams(**vals)

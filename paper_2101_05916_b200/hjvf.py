"""HJVF value-field container (reference proj/include/hjsafe/hjvf.hpp:10-13,
proj/src/hjvf.cpp:46-95), little-endian:

    magic "HJVF" | version u32 (=1) | ndims u32 | per dim {n u64, min f64, max f64}
    | values f64, row-major, last dim fastest

Round-trips bit-exactly.  Readers reject bad magic, versions other than 1,
ndims outside 1..32, truncated streams and non-finite values, as the
reference does.
"""
from __future__ import annotations

import struct
from pathlib import Path

import numpy as np

from . import hjsafe as hj

MAGIC = b"HJVF"
VERSION = 1


def dumps(field: hj.ScalarField) -> bytes:
    g = field.grid()
    out = [MAGIC, struct.pack("<II", VERSION, g.ndims())]
    for d in g.dims():
        out.append(struct.pack("<Qdd", d.n, d.min, d.max))
    out.append(np.ascontiguousarray(field.values(), dtype="<f8").tobytes())
    return b"".join(out)


def loads(data: bytes) -> hj.ScalarField:
    if len(data) < 12 or data[:4] != MAGIC:
        raise RuntimeError("HJVF: bad magic")
    version, ndims = struct.unpack_from("<II", data, 4)
    if version != VERSION:
        raise RuntimeError(f"HJVF: unsupported version {version}")
    if ndims == 0 or ndims > 32:
        raise RuntimeError("HJVF: bad ndims")
    off = 12
    dims = []
    for _ in range(ndims):
        if off + 24 > len(data):
            raise RuntimeError("HJVF: truncated stream")
        n, lo, hi = struct.unpack_from("<Qdd", data, off)
        dims.append((lo, hi, n))
        off += 24
    grid = hj.Grid(dims)
    need = grid.size() * 8
    if off + need > len(data):
        raise RuntimeError("HJVF: truncated stream")
    v = np.frombuffer(data, dtype="<f8", count=grid.size(), offset=off).astype(np.float64)
    if not np.all(np.isfinite(v)):
        raise RuntimeError("HJVF: non-finite value")
    return hj.ScalarField(grid, v)


def write(path, field: hj.ScalarField) -> None:
    Path(path).write_bytes(dumps(field))


def read(path) -> hj.ScalarField:
    return loads(Path(path).read_bytes())

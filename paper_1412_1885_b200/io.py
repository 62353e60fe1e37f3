"""The reference's binary model/tensor files (io.hpp:52-183), so models and data move
between tenkit tooling and this library: little-endian, f64, column-major.

  .dten  "DTEN" u32 version=1, u32 order, u32 dims[order], f64 payload
  .tkr   "TKRM" u32 1, u32 order, u32 core dims[order], (u32 rows, u32 cols)[order],
         f64 core, f64 factors in mode order
  .cpm   "CPMD" u32 1, u32 order, u32 rank, u32 dims[order], f64 factors in mode order

Errors raise TenkitIOError("tenkit io: ...") where the reference throws
std::runtime_error (io.hpp:16-18). load_dten(..., dtype=np.float32) converts in chunks so a
large fp64 file becomes the fp32 workload without a full fp64 copy in memory.
"""
from __future__ import annotations

import struct

import numpy as np

from .tenkit import CpModel, DenseTensor, TuckerModel


class TenkitIOError(RuntimeError):
    pass


def _check(ok: bool, msg: str):
    if not ok:
        raise TenkitIOError("tenkit io: " + msg)


def _u32(f) -> int:
    b = f.read(4)
    _check(len(b) == 4, "unexpected end of file")
    return struct.unpack("<I", b)[0]


def _magic(f, magic: bytes, what: str):
    b = f.read(4)
    _check(b == magic, f"bad magic for {what} file")
    _check(_u32(f) == 1, f"unsupported {what} file version")


def _f64(f, n: int) -> np.ndarray:
    a = np.empty(n, dtype="<f8")
    got = f.readinto(memoryview(a).cast("B")) if n else 0
    _check(got == 8 * n, "unexpected end of file")
    return a


def _host(x) -> np.ndarray:
    if hasattr(x, "detach"):
        x = x.detach().cpu().numpy()
    return np.asarray(x, dtype=np.float64)


# ------------------------------------------------------------------------------- .dten
def write_dten(f, t) -> None:
    """t: DenseTensor (host or device) or a numpy n-d array (column-major semantics)."""
    if isinstance(t, DenseTensor):
        shape, flat = t.shape, _host(t.data).ravel()
    else:
        a = np.asarray(t)
        shape, flat = a.shape, a.astype(np.float64).ravel(order="F")
    f.write(b"DTEN" + struct.pack("<II", 1, len(shape)) + struct.pack(f"<{len(shape)}I", *shape))
    f.write(np.ascontiguousarray(flat, dtype="<f8").tobytes())


def read_dten(f, dtype=np.float64, chunk: int = 1 << 26) -> DenseTensor:
    _magic(f, b"DTEN", "tensor")
    order = _u32(f)
    _check(order >= 1, "tensor order must be positive")
    shape = tuple(_u32(f) for _ in range(order))
    n = int(np.prod(shape))
    if np.dtype(dtype) == np.float64:
        return DenseTensor(shape, _f64(f, n))
    out = np.empty(n, dtype=dtype)
    for a in range(0, n, chunk):
        m = min(chunk, n - a)
        out[a:a + m] = _f64(f, m)
    return DenseTensor(shape, out)


# ------------------------------------------------------------------------------- .tkr
def write_tkr(f, model: TuckerModel) -> None:
    m = model.to_host()
    core = np.asarray(m.core, dtype=np.float64)
    cshape = core.shape if core.ndim == len(m.factors) else tuple(m.core_shape)
    fs = [np.asarray(u, dtype=np.float64) for u in m.factors]
    _check(len(fs) == len(cshape), "tucker model: one factor per mode required")
    for n, u in enumerate(fs):
        _check(u.ndim == 2 and u.shape[1] == cshape[n], "tucker model: factor columns must match core shape")
    f.write(b"TKRM" + struct.pack("<II", 1, len(cshape)) + struct.pack(f"<{len(cshape)}I", *cshape))
    for u in fs:
        f.write(struct.pack("<II", *u.shape))
    f.write(np.ascontiguousarray(core.ravel(order="F"), dtype="<f8").tobytes())
    for u in fs:
        f.write(np.ascontiguousarray(u.ravel(order="F"), dtype="<f8").tobytes())


def read_tkr(f) -> TuckerModel:
    _magic(f, b"TKRM", "tucker model")
    order = _u32(f)
    _check(order >= 1, "model order must be positive")
    cshape = tuple(_u32(f) for _ in range(order))
    fd = [(_u32(f), _u32(f)) for _ in range(order)]
    core = _f64(f, int(np.prod(cshape))).reshape(cshape, order="F")
    fs = [_f64(f, r * c).reshape((r, c), order="F") for r, c in fd]
    for n, (r, c) in enumerate(fd):
        _check(c == cshape[n], "tucker model: factor columns must match core shape")
    return TuckerModel(core, fs, cshape)


# ------------------------------------------------------------------------------- .cpm
def write_cpm(f, model) -> None:
    fs = [_host(a) for a in (model.factors if hasattr(model, "factors") else model)]
    _check(len(fs) >= 1, "cp model: no factors")
    rank = fs[0].shape[1]
    _check(rank >= 1 and all(a.ndim == 2 and a.shape[1] == rank for a in fs), "cp model: factor rank mismatch")
    f.write(b"CPMD" + struct.pack("<III", 1, len(fs), rank) + struct.pack(f"<{len(fs)}I", *[a.shape[0] for a in fs]))
    for a in fs:
        f.write(np.ascontiguousarray(a.ravel(order="F"), dtype="<f8").tobytes())


def read_cpm(f) -> CpModel:
    _magic(f, b"CPMD", "cp model")
    order = _u32(f)
    rank = _u32(f)
    _check(order >= 1 and rank >= 1, "invalid cp model header")
    dims = [_u32(f) for _ in range(order)]
    return CpModel([_f64(f, d * rank).reshape((d, rank), order="F") for d in dims])


# ------------------------------------------------------------------------------- paths
def _open(path, mode):
    try:
        return open(path, mode)
    except OSError:
        raise TenkitIOError(f"tenkit io: cannot open {path}" + (" for writing" if "w" in mode else "")) from None


def save_dten(path, t):
    with _open(path, "wb") as f:
        write_dten(f, t)


def save_tkr(path, m):
    with _open(path, "wb") as f:
        write_tkr(f, m)


def save_cpm(path, m):
    with _open(path, "wb") as f:
        write_cpm(f, m)


def load_dten(path, dtype=np.float64) -> DenseTensor:
    with _open(path, "rb") as f:
        return read_dten(f, dtype)


def load_tkr(path) -> TuckerModel:
    with _open(path, "rb") as f:
        return read_tkr(f)


def load_cpm(path) -> CpModel:
    with _open(path, "rb") as f:
        return read_cpm(f)

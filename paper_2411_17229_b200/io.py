"""Reference artifact formats (proj/docs/FILE_FORMATS.md) — the interchange
boundary between a GPU-built index and the reference CPU library.

DADE transform  proj/src/transform.cpp:306-358
.cal table      proj/src/calibration.cpp:184-212
DIVF index      proj/src/ivf.cpp:233-279 (contiguous layout writes split = D)
fvecs / ivecs   proj/src/dataset_io.cpp:36-99
"""
from __future__ import annotations

import struct
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from .api import CalibrationTable, OrthoTransform


@dataclass
class Divf:
    dim: int
    count: int
    n_clusters: int
    layout: int
    split: int
    centroids: np.ndarray  # [C, D] f32
    offsets: np.ndarray    # [C+1] u32
    ids: np.ndarray        # [N] u32
    storage: np.ndarray    # [N*D] f32 (layout as stored)


def write_divf(path, d: Divf) -> None:
    with open(path, "wb") as f:
        f.write(b"DIVF")
        f.write(struct.pack("<IBIIII", 1, d.layout, d.dim, d.count, d.n_clusters, d.split))
        f.write(np.ascontiguousarray(d.centroids, "<f4").tobytes())
        f.write(np.ascontiguousarray(d.offsets, "<u4").tobytes())
        f.write(np.ascontiguousarray(d.ids, "<u4").tobytes())
        f.write(np.ascontiguousarray(d.storage, "<f4").tobytes())


def read_divf(path) -> Divf:
    b = Path(path).read_bytes()
    if b[:4] != b"DIVF":
        raise RuntimeError(f"not an ivf index file: {path}")
    ver, layout, dim, count, nc, split = struct.unpack_from("<IBIIII", b, 4)
    if ver != 1:
        raise RuntimeError(f"unsupported ivf index version {ver}")
    if layout > 1:
        raise RuntimeError("bad ivf layout byte")
    if dim == 0 or nc == 0 or split == 0 or split > dim:
        raise RuntimeError("inconsistent ivf header")
    off = 25
    need = off + 4 * (nc * dim + nc + 1 + count + count * dim)
    if len(b) < need:
        raise RuntimeError("truncated file while reading ivf payload")
    cen = np.frombuffer(b, "<f4", nc * dim, off).reshape(nc, dim).copy(); off += 4 * nc * dim
    offs = np.frombuffer(b, "<u4", nc + 1, off).copy(); off += 4 * (nc + 1)
    if offs[0] != 0 or offs[-1] != count or np.any(np.diff(offs.astype(np.int64)) < 0):
        raise RuntimeError("inconsistent ivf posting offsets")
    ids = np.frombuffer(b, "<u4", count, off).copy(); off += 4 * count
    sto = np.frombuffer(b, "<f4", count * dim, off).copy()
    return Divf(dim, count, nc, layout, split, cen, offs, ids, sto)


def write_transform(path, t: OrthoTransform) -> None:
    with open(path, "wb") as f:
        f.write(b"DADE")
        f.write(struct.pack("<IBI", 1, t.kind, t.dim))
        f.write(np.ascontiguousarray(t.mean, "<f8").tobytes())
        f.write(np.ascontiguousarray(t.eigenvalues, "<f8").tobytes())
        f.write(np.ascontiguousarray(t.matrix, "<f8").tobytes())


def read_transform(path) -> OrthoTransform:
    b = Path(path).read_bytes()
    if b[:4] != b"DADE":
        raise RuntimeError(f"not a transform file: {path}")
    ver, kind, dim = struct.unpack_from("<IBI", b, 4)
    if ver != 1:
        raise RuntimeError(f"unsupported transform version {ver}")
    if kind > 1:
        raise RuntimeError("bad transform kind byte")
    if dim == 0:
        raise RuntimeError("transform dim is zero")
    off = 13
    mean = np.frombuffer(b, "<f8", dim, off).copy(); off += 8 * dim
    ev = np.frombuffer(b, "<f8", dim, off).copy(); off += 8 * dim
    mat = np.frombuffer(b, "<f8", dim * dim, off).copy()
    if len(b) < off + 8 * dim * dim:
        raise RuntimeError("truncated file while reading matrix")
    if np.any(ev[:-1] < ev[1:]):
        raise RuntimeError("transform eigenvalues not nonincreasing")
    # the loader's corruption check (proj/src/transform.cpp:344-356): columns orthonormal
    cols = mat.reshape(dim, dim)  # row k = column k of the column-major matrix
    worst = float(np.max(np.abs(cols @ cols.T - np.eye(dim))))
    if worst > 1e-5:
        raise RuntimeError(f"transform matrix not orthogonal (max deviation {worst:.6f})")
    return OrthoTransform(dim, kind, mean, ev, mat)


def write_cal(path, c: CalibrationTable) -> None:
    with open(path, "wb") as f:
        f.write(struct.pack("<dII", c.p_s, c.delta_d, len(c.checkpoints)))
        for d, e in zip(c.checkpoints, c.epsilons):
            f.write(struct.pack("<Id", d, e))


def read_cal(path) -> CalibrationTable:
    b = Path(path).read_bytes()
    p_s, dd, n = struct.unpack_from("<dII", b, 0)
    cps, eps = [], []
    for i in range(n):
        d, e = struct.unpack_from("<Id", b, 16 + 12 * i)
        cps.append(d)
        eps.append(e)
    if any(cps[i] >= cps[i + 1] for i in range(n - 1)):
        raise RuntimeError("calibration checkpoints not ascending")
    return CalibrationTable(p_s, dd, cps, eps)


def write_fvecs(path, a: np.ndarray) -> None:
    a = np.ascontiguousarray(a, "<f4")
    n, d = a.shape
    rec = np.empty((n, d + 1), "<f4")
    rec[:, 0] = np.frombuffer(np.int32(d).tobytes(), "<f4")[0]
    rec[:, 1:] = a
    Path(path).write_bytes(rec.tobytes())


def read_fvecs(path) -> np.ndarray:
    raw = np.fromfile(path, "<i4")
    d = int(raw[0])
    return raw.reshape(-1, d + 1)[:, 1:].view("<f4").copy()


def write_ivecs(path, a: np.ndarray) -> None:
    a = np.ascontiguousarray(a, "<i4")
    n, d = a.shape
    rec = np.empty((n, d + 1), "<i4")
    rec[:, 0] = d
    rec[:, 1:] = a
    Path(path).write_bytes(rec.tobytes())


def read_ivecs(path) -> np.ndarray:
    raw = np.fromfile(path, "<i4")
    d = int(raw[0])
    return raw.reshape(-1, d + 1)[:, 1:].copy()

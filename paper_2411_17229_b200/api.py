"""Python mirror of the reference's search API over the C ABI.

Names, argument meaning and error behaviour follow proj/include/dade/*.hpp:
``OrthoTransform``, ``CalibrationTable``, ``FdScanningStrategy``,
``DadeStrategy``, ``AdsamplingStrategy``, ``IvfIndex.search``,
``linear_scan``, ``DcoStats``, ``SearchResult``; batched variants
(``search_batch``) are the GPU-native granularity. Every compute call goes to
libdade_gpu.so; there is no host fallback.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field

import numpy as np

from . import _capi
from ._capi import ConfigError, InvalidInput, check, ptr

__all__ = [
    "Device", "OrthoTransform", "CalibrationTable", "FdScanningStrategy", "DadeStrategy",
    "AdsamplingStrategy", "IvfIndex", "FlatIndex", "linear_scan", "DcoStats", "DcoOutcome",
    "SearchResult", "Neighbor", "ConfigError", "InvalidInput", "expected_checkpoints",
    "compute_covariance", "fit_pca", "kmeans", "compute_ground_truth",
]


def _f32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float32)


def _u32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.uint32)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def expected_checkpoints(dim: int, delta_d: int) -> list[int]:
    """CalibrationTable::expected_checkpoints (proj/src/calibration.cpp:74-81)."""
    if delta_d == 0:
        raise InvalidInput("delta_d must be positive")
    return list(range(delta_d, dim, delta_d))


class Device:
    """One GPU context (dade_gpu_ctx): owns device copies of the artifacts."""

    def __init__(self, device: int = 0):
        h = C.c_void_p()
        check(_capi.lib.dade_gpu_create(device, C.byref(h)))
        self.h = h
        self.device = device
        self._strategy_token = None

    def close(self):
        if self.h:
            _capi.lib.dade_gpu_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_stream(self, stream_ptr: int | None):
        check(_capi.lib.dade_gpu_set_stream(self.h, C.c_void_p(stream_ptr)))

    def synchronize(self):
        check(_capi.lib.dade_gpu_synchronize(self.h))

    @property
    def launches(self) -> int:
        return int(_capi.lib.dade_gpu_launch_count(self.h))

    def set_profiling(self, on: bool):
        check(_capi.lib.dade_gpu_set_profiling(self.h, int(on)))

    def set_graphs(self, on: bool):
        """Replay captured CUDA graphs of repeated IVF searches (default on)."""
        check(_capi.lib.dade_gpu_set_graphs(self.h, int(on)))

    def last_filter_profile(self):
        ms, n = C.c_double(), C.c_int()
        check(_capi.lib.dade_gpu_last_filter_profile(self.h, C.byref(ms), C.byref(n)))
        return ms.value, n.value

    def last_seed_profile(self):
        ms, pd = C.c_double(), C.c_double()
        check(_capi.lib.dade_gpu_last_seed_profile(self.h, C.byref(ms), C.byref(pd)))
        return ms.value, pd.value

    def last_union_profile(self):
        """(B_union bytes, rows touched) of the last profiled streaming search."""
        a, b = C.c_double(), C.c_double()
        check(_capi.lib.dade_gpu_last_union_profile(self.h, C.byref(a), C.byref(b)))
        return a.value, b.value

    def last_scan_profile(self):
        a, b, c = C.c_double(), C.c_double(), C.c_double()
        check(_capi.lib.dade_gpu_last_scan_profile(self.h, C.byref(a), C.byref(b), C.byref(c)))
        return a.value, b.value, c.value

    def set_estimate_dump(self, capacity: int):
        """Record every checkpoint partial the hot path evaluates (0 disables)."""
        check(_capi.lib.dade_gpu_set_estimate_dump(self.h, int(capacity)))

    def estimate_dump(self, cap: int):
        """(query, id, d, partial f32, estimate f64) arrays of the last search's
        evaluated checkpoints, and the number recorded."""
        q = np.zeros(cap, np.uint32)
        ids = np.zeros(cap, np.uint32)
        dims = np.zeros(cap, np.uint32)
        part = np.zeros(cap, np.float32)
        est = np.zeros(cap, np.float64)
        n = C.c_uint64()
        check(_capi.lib.dade_gpu_get_estimate_dump(self.h, cap, ptr(q), ptr(ids), ptr(dims), ptr(part), ptr(est),
                                                   C.byref(n)))
        m = min(int(n.value), cap)
        return (q[:m], ids[:m], dims[:m], part[:m], est[:m]), int(n.value)

    # -- strategy plumbing ---------------------------------------------------
    def apply(self, dco) -> None:
        if self._strategy_token is dco:
            return
        dco._apply(self)
        self._strategy_token = dco


@dataclass
class OrthoTransform:
    """proj/include/dade/transform.hpp:42-64 (column-major f64 matrix)."""
    dim: int
    kind: int  # 0 pca, 1 random
    mean: np.ndarray
    eigenvalues: np.ndarray
    matrix: np.ndarray  # D*D column-major (column k = k-th direction)

    @property
    def lambda_prefix(self) -> np.ndarray:
        ev = np.maximum(self.eigenvalues, 0.0)
        out = np.zeros(self.dim + 1)
        acc = 0.0
        for i, v in enumerate(ev):  # sequential sums, as prefix_sums()
            acc = acc + float(v)
            out[i + 1] = acc
        return out

    def scale_factor(self, d: int) -> float:
        """OrthoTransform::scale_factor (proj/src/transform.cpp:209-214)."""
        if d == 0 or d > self.dim:
            raise InvalidInput("scale_factor: d out of range")
        pre = self.lambda_prefix
        return 1.0 if pre[d] <= 0.0 else pre[self.dim] / pre[d]

    def upload(self, dev: Device):
        check(_capi.lib.dade_gpu_set_transform(dev.h, self.dim, ptr(_f64(self.matrix)),
                                               ptr(_f64(self.eigenvalues))))

    def apply(self, dev: Device, rows: np.ndarray) -> np.ndarray:
        """apply_transform (proj/src/transform.cpp:295-304) on the GPU."""
        rows = _f32(rows)
        if rows.ndim != 2 or rows.shape[1] != self.dim:
            raise InvalidInput("apply_transform: dimension mismatch")
        self.upload(dev)
        out = np.empty_like(rows)
        check(_capi.lib.dade_gpu_rotate(dev.h, ptr(rows), rows.shape[0], ptr(out), 0))
        return out


@dataclass
class CalibrationTable:
    """proj/include/dade/calibration.hpp:20-40."""
    p_s: float
    delta_d: int
    checkpoints: list
    epsilons: list

    @staticmethod
    def expected_checkpoints(dim: int, delta_d: int) -> list[int]:
        return expected_checkpoints(dim, delta_d)

    @staticmethod
    def unbounded(dim: int, delta_d: int) -> "CalibrationTable":
        cps = expected_checkpoints(dim, delta_d)
        return CalibrationTable(0.0, delta_d, cps, [math.inf] * len(cps))

    @staticmethod
    def calibrate(dev: Device, t: OrthoTransform, transformed_data, p_s: float, delta_d: int,
                  n_pairs: int, seed: int, device_ptr: bool = False, count: int | None = None):
        """calibrate (proj/src/calibration.cpp:109-146), partial sums on the GPU.
        With device_ptr, ``transformed_data`` is a CUDA tensor [count, dim]."""
        t.upload(dev)
        n = count if count is not None else int(transformed_data.shape[0])
        data = transformed_data if device_ptr else _f32(transformed_data)
        cps = np.zeros(max(1, t.dim // max(delta_d, 1) + 1), dtype=np.uint32)
        eps = np.zeros(len(cps), dtype=np.float64)
        nout = C.c_uint32()
        check(_capi.lib.dade_gpu_calibrate(dev.h, ptr(data), n, float(p_s), delta_d, int(n_pairs),
                                           int(seed), _capi.DEVICE_PTRS if device_ptr else 0,
                                           ptr(cps), ptr(eps), C.byref(nout)))
        m = nout.value
        return CalibrationTable(float(p_s), delta_d, [int(x) for x in cps[:m]],
                                [float(x) for x in eps[:m]])


class _Strategy:
    kind = _capi.FD
    dim = 0

    @property
    def n_ckpt(self) -> int:
        if isinstance(self, DadeStrategy):
            return len(self.cal.checkpoints)
        if isinstance(self, AdsamplingStrategy):
            return len(expected_checkpoints(self.dim, self.delta_d))
        return 0


class FdScanningStrategy(_Strategy):
    """proj/src/estimator.cpp:99-113: exact distance, prune iff > r."""
    kind = _capi.FD

    def __init__(self, dim: int):
        self.dim = dim
        self.checkpoints, self.reject_coeff, self.est_scale = [], [], []

    def _apply(self, dev: Device):
        check(_capi.lib.dade_gpu_set_strategy(dev.h, _capi.FD, self.dim, 0, None, None, None))


class DadeStrategy(_Strategy):
    """DadeStrategy(t, cal, delta_d) (proj/src/estimator.cpp:115-152); the
    table derivation and its ConfigError checks run in the C ABI."""
    kind = _capi.DADE

    def __init__(self, t: OrthoTransform, cal: CalibrationTable, delta_d: int, dev: Device | None = None):
        self.t, self.cal, self.delta_d, self.dim = t, cal, delta_d, t.dim
        self._dev = dev or _default_device()
        self._apply(self._dev)  # validate eagerly, like the reference ctor
        self._dev._strategy_token = self

    def _apply(self, dev: Device):
        self.t.upload(dev)
        cps = _u32(self.cal.checkpoints)
        eps = _f64(self.cal.epsilons)
        check(_capi.lib.dade_gpu_set_strategy_dade(dev.h, self.delta_d, self.cal.delta_d, len(cps),
                                                   ptr(cps), ptr(eps)))


class AdsamplingStrategy(_Strategy):
    """proj/src/estimator.cpp:158-177."""
    kind = _capi.ADS

    def __init__(self, dim: int, delta_d: int, eps0: float, dev: Device | None = None):
        self.dim, self.delta_d, self.eps0 = dim, delta_d, eps0
        d = dev or _default_device()
        self._apply(d)
        d._strategy_token = self

    def _apply(self, dev: Device):
        check(_capi.lib.dade_gpu_set_strategy_ads(dev.h, self.dim, self.delta_d, float(self.eps0)))


_DEFAULT = None


def _default_device() -> Device:
    global _DEFAULT
    if _DEFAULT is None:
        _DEFAULT = Device(0)
    return _DEFAULT


@dataclass
class DcoStats:
    """proj/include/dade/estimator.hpp:24-49."""
    total_dco: int = 0
    dims_accumulated: int = 0
    measure_failures: bool = False
    eligible: int = 0
    failures: int = 0

    def _add(self, s: _capi.Stats):
        self.total_dco += s.total_dco
        self.dims_accumulated += s.dims_accumulated
        self.eligible += s.eligible
        self.failures += s.failures

    def dim_fraction(self, dim: int) -> float:
        return 0.0 if self.total_dco == 0 else self.dims_accumulated / (self.total_dco * dim)

    def failure_rate(self) -> float:
        return 0.0 if self.eligible == 0 else self.failures / self.eligible


@dataclass
class DcoOutcome:
    pruned: bool
    distance: float
    distance_exact: bool
    dims_used: int


@dataclass(order=True)
class Neighbor:
    distance: float
    id: int


@dataclass
class SearchResult:
    neighbors: list = field(default_factory=list)
    truncated: bool = False

    def ids(self):
        return [n.id for n in self.neighbors]


def _results(ids, dists, counts, k):
    out = []
    for q in range(ids.shape[0]):
        c = int(counts[q])
        out.append(SearchResult([Neighbor(float(dists[q, i]), int(ids[q, i])) for i in range(c)], c < k))
    return out


def evaluate_batch(dev: Device, dco, o, q, r, stats: DcoStats | None = None):
    """DcoStrategy::evaluate over n independent (o_i, q_i, r_i) on the GPU."""
    dev.apply(dco)
    o, q, r = _f32(o), _f32(q), _f32(np.atleast_1d(r))
    n = r.shape[0]
    pr = np.zeros(n, np.uint8)
    di = np.zeros(n, np.float32)
    ex = np.zeros(n, np.uint8)
    du = np.zeros(n, np.uint32)
    st = _capi.Stats()
    check(_capi.lib.dade_gpu_dco_evaluate(dev.h, ptr(o), ptr(q), ptr(r), n, 0, ptr(pr), ptr(di),
                                          ptr(ex), ptr(du), C.byref(st)))
    if stats is not None:
        stats.total_dco += st.total_dco
        stats.dims_accumulated += st.dims_accumulated
        if stats.measure_failures:
            stats.eligible += st.eligible
            stats.failures += st.failures
    return pr.astype(bool), di, ex.astype(bool), du


def partial_sums(dev: Device, dco, o, q) -> np.ndarray:
    """Running partial squared distances at each checkpoint and at dim."""
    dev.apply(dco)
    o, q = _f32(o), _f32(q)
    n = o.shape[0]
    out = np.zeros((n, dco.n_ckpt + 1), np.float32)
    check(_capi.lib.dade_gpu_partial_sums(dev.h, ptr(o), ptr(q), n, 0, ptr(out)))
    return out


class IvfIndex:
    """Device-resident IVF index in the reference's DIVF field order
    (proj/include/dade/ivf.hpp:62-70; proj/src/ivf.cpp:233-279)."""

    def __init__(self, dev: Device, dim, count, n_clusters, centroids, offsets, ids, storage,
                 layout: int = 0, split: int | None = None):
        self.dev = dev
        self._dim, self._count, self._nc = int(dim), int(count), int(n_clusters)
        self.layout = layout
        self.split = dim if split is None else split
        self.offsets = _u32(offsets)
        check(_capi.lib.dade_gpu_set_ivf(dev.h, self._dim, self._count, self._nc, layout, self.split,
                                         ptr(_f32(centroids)), ptr(self.offsets), ptr(_u32(ids)),
                                         ptr(_f32(storage))))

    @staticmethod
    def build(dev: Device, data, n_clusters: int, kmeans_max_iters: int, seed: int) -> "IvfIndex":
        """IvfIndex::build (proj/src/ivf.cpp:145-192, contiguous layout) on the
        GPU; the DIVF arrays are on the returned index (centroids, offsets, ids,
        storage), equal to the reference's."""
        x = _rows(data)
        n, d = int(x.shape[0]), int(x.shape[1])
        cen = np.zeros((n_clusters, d), np.float32)
        off = np.zeros(n_clusters + 1, np.uint32)
        ids = np.zeros(n, np.uint32)
        sto = np.zeros((n, d), np.float32)
        check(_capi.lib.dade_gpu_ivf_build(dev.h, ptr(x), n, d, n_clusters, kmeans_max_iters, int(seed),
                                           _dev_flag(x), ptr(cen), ptr(off), ptr(ids), ptr(sto)))
        idx = IvfIndex.__new__(IvfIndex)
        idx.dev, idx._dim, idx._count, idx._nc = dev, d, n, n_clusters
        idx.layout, idx.split, idx.offsets = 0, d, off
        idx.centroids, idx.ids, idx.storage = cen, ids, sto
        return idx

    @staticmethod
    def from_divf(dev: Device, divf) -> "IvfIndex":
        return IvfIndex(dev, divf.dim, divf.count, divf.n_clusters, divf.centroids, divf.offsets,
                        divf.ids, divf.storage, divf.layout, divf.split)

    def dim(self):
        return self._dim

    def count(self):
        return self._count

    def n_clusters(self):
        return self._nc

    def shard(self, list_mask) -> None:
        m = np.ascontiguousarray(list_mask, dtype=np.uint8)
        check(_capi.lib.dade_gpu_set_ivf_shard(self.dev.h, ptr(m)))

    def search_batch(self, queries, k: int, n_probe: int, dco, stats: DcoStats | None = None,
                     raw: bool = False):
        """Batched IvfIndex::search; returns (ids [nq,k], dists [nq,k], counts [nq])."""
        q = _f32(queries)
        if q.ndim == 1:
            q = q[None, :]
        if q.shape[1] != self._dim:
            raise InvalidInput("IvfIndex::search: query dim mismatch")
        if dco.dim != self._dim:
            raise InvalidInput("IvfIndex::search: strategy dim mismatch")
        self.dev.apply(dco)
        nq = q.shape[0]
        kk = max(k, 1)
        ids = np.zeros((nq, kk), np.uint32)
        dists = np.zeros((nq, kk), np.float32)
        counts = np.zeros(nq, np.uint32)
        st = _capi.Stats()
        flags = (_capi.QUERIES_RAW if raw else 0) | (_capi.MEASURE_FAILURES if stats and stats.measure_failures else 0)
        check(_capi.lib.dade_gpu_ivf_search(self.dev.h, ptr(q), nq, k, n_probe, flags, ptr(ids), ptr(dists),
                                            ptr(counts), C.byref(st)))
        if stats is not None:
            stats._add(st)
        return ids, dists, counts

    def search_batches(self, batches, k: int, n_probe: int, dco, stats: DcoStats | None = None,
                       raw: bool = False, outputs=None):
        """A sequence of equal-sized query batches searched with the copies of
        one batch under the search of its neighbours (dade_gpu_ivf_search_batches);
        results identical to search_batch per batch. outputs: optional list of
        (ids, dists, counts) arrays to fill (pinned host memory overlaps best).
        Returns the list of (ids, dists, counts)."""
        qs = [_f32(b) for b in batches]
        if not qs:
            return []
        nq = qs[0].shape[0]
        for q in qs:
            if q.ndim != 2 or q.shape != (nq, self._dim):
                raise InvalidInput("IvfIndex::search: every batch must be [nq, dim]")
        if dco.dim != self._dim:
            raise InvalidInput("IvfIndex::search: strategy dim mismatch")
        self.dev.apply(dco)
        kk = max(k, 1)
        if outputs is None:
            outputs = [(np.zeros((nq, kk), np.uint32), np.zeros((nq, kk), np.float32), np.zeros(nq, np.uint32))
                       for _ in qs]
        if len(outputs) != len(qs):
            raise InvalidInput("IvfIndex::search: one (ids, dists, counts) output per batch")
        want = (((nq, kk), np.uint32), ((nq, kk), np.float32), ((nq,), np.uint32))
        for out in outputs:  # the C ABI writes nq*k*4 bytes through each pointer
            if len(out) != 3:
                raise InvalidInput("IvfIndex::search: outputs are (ids, dists, counts) triples")
            for a, (shape, dt) in zip(out, want):
                ok = (isinstance(a, np.ndarray) and a.flags.c_contiguous and a.shape == shape and a.dtype == dt) or \
                     (hasattr(a, "data_ptr") and a.is_contiguous() and tuple(a.shape) == shape and
                      a.element_size() == 4 and a.device.type == "cpu")
                if not ok:
                    raise InvalidInput(f"IvfIndex::search: output must be a C-contiguous host array of shape "
                                       f"{shape} and dtype {np.dtype(dt).name}")
        nb = len(qs)
        PA = C.c_void_p * nb
        st = _capi.Stats()
        check(_capi.lib.dade_gpu_ivf_search_batches(
            self.dev.h, nb, PA(*[ptr(q) for q in qs]), nq, k, n_probe, _capi.QUERIES_RAW if raw else 0,
            PA(*[ptr(o[0]) for o in outputs]), PA(*[ptr(o[1]) for o in outputs]),
            PA(*[ptr(o[2]) for o in outputs]), C.byref(st)))
        if stats is not None:
            stats._add(st)
        return outputs

    def search(self, query, k: int, n_probe: int, dco, stats: DcoStats | None = None) -> SearchResult:
        """IvfIndex::search (proj/src/ivf.cpp:207-231) for one rotated query."""
        ids, dists, counts = self.search_batch(query, k, n_probe, dco, stats)
        return _results(ids, dists, counts, k)[0]

    def search_many(self, queries, k, n_probe, dco, stats=None):
        ids, dists, counts = self.search_batch(queries, k, n_probe, dco, stats)
        return _results(ids, dists, counts, k)


class FlatIndex:
    """Device-resident base rows for linear_scan (proj/src/knn.cpp:31-41)."""

    def __init__(self, dev: Device, data, id_base: int = 0):
        self.dev = dev
        d = _f32(data)
        if d.ndim != 2 or d.shape[1] == 0:
            raise InvalidInput("VectorSet: dim must be positive")
        self.dim, self.count = d.shape[1], d.shape[0]
        self.parts = 0
        check(_capi.lib.dade_gpu_set_base(dev.h, self.dim, self.count, ptr(d), id_base))

    def partition(self, n_parts: int, max_iters: int = 10, seed: int = 1):
        """Data-ordered scan (dade_gpu_flat_partition): k-means cells of the base
        on the GPU become the visiting order (every cell probed, each query's
        nearest first). Replaces the Device's IVF index; 0 drops it."""
        check(_capi.lib.dade_gpu_flat_partition(self.dev.h, int(n_parts), int(max_iters), int(seed)))
        self.parts = int(n_parts)
        return self

    def search_batch(self, queries, k: int, dco, stats: DcoStats | None = None, raw: bool = False):
        q = _f32(queries)
        if q.ndim == 1:
            q = q[None, :]
        if dco.dim != self.dim:
            raise InvalidInput("linear_scan: strategy dim mismatch")
        self.dev.apply(dco)
        nq = q.shape[0]
        kk = max(k, 1)
        ids = np.zeros((nq, kk), np.uint32)
        dists = np.zeros((nq, kk), np.float32)
        counts = np.zeros(nq, np.uint32)
        st = _capi.Stats()
        flags = (_capi.QUERIES_RAW if raw else 0) | (_capi.MEASURE_FAILURES if stats and stats.measure_failures else 0)
        check(_capi.lib.dade_gpu_flat_search(self.dev.h, ptr(q), nq, k, flags, ptr(ids), ptr(dists), ptr(counts),
                                             C.byref(st)))
        if stats is not None:
            stats._add(st)
        return ids, dists, counts


# ---- index build on the GPU, reference arithmetic ---------------

def _dev_flag(x) -> int:
    return _capi.DEVICE_PTRS if hasattr(x, "data_ptr") and getattr(x, "is_cuda", False) else 0


def _rows(x):
    """numpy -> C-contiguous f32; CUDA tensors pass through (device pointers)."""
    if hasattr(x, "data_ptr") and getattr(x, "is_cuda", False):
        assert x.dtype.itemsize == 4 and x.is_contiguous() and x.dim() == 2
        return x
    return _f32(x)


def compute_covariance(dev: Device, data):
    """compute_covariance (proj/src/transform.cpp:68-95) on the GPU: (mean [D],
    cov [D, D]) bit-identical to the reference."""
    x = _rows(data)
    n, d = int(x.shape[0]), int(x.shape[1])
    mean = np.zeros(d, np.float64)
    cov = np.zeros((d, d), np.float64)
    check(_capi.lib.dade_gpu_covariance(dev.h, ptr(x), n, d, _dev_flag(x), ptr(mean), ptr(cov)))
    return mean, cov


def fit_pca(dev: Device, data) -> OrthoTransform:
    """fit_pca (proj/src/transform.cpp:230-253): covariance on the GPU (exact),
    symmetric eigendecomposition in fp64 (LAPACK; the reference runs cyclic
    Jacobi, equal to ~1e-12 relative on the well-separated spectra used here),
    then the reference's column order (variance descending, stable on ties),
    orientation (first nonzero component positive) and eigenvalue clamp."""
    mean, cov = compute_covariance(dev, data)
    d = cov.shape[0]
    vals, vecs = np.linalg.eigh(cov)
    order = sorted(range(d), key=lambda i: -vals[i])  # stable: original position on ties
    eig = np.array([vals[i] for i in order])
    cols = np.stack([vecs[:, i] for i in order])  # row k = k-th direction
    for k in range(d):  # orient_column
        nz = np.nonzero(cols[k])[0]
        if nz.size and cols[k, nz[0]] < 0:
            cols[k] = -cols[k]
    if np.any(eig < -1e-6):
        raise RuntimeError("eigenvalue below tolerance; input is not positive semidefinite")
    eig = np.where(eig < 0.0, 0.0, eig)
    return OrthoTransform(d, 0, mean, eig, np.ascontiguousarray(cols).reshape(-1))


def kmeans(dev: Device, data, n_clusters: int, max_iters: int, seed: int):
    """kmeans (proj/src/ivf.cpp:24-143) on the GPU: (centroids [C, D],
    assignments [N], iterations), equal to the reference's."""
    x = _rows(data)
    n, d = int(x.shape[0]), int(x.shape[1])
    cen = np.zeros((n_clusters, d), np.float32)
    asg = np.zeros(n, np.uint32)
    it = C.c_uint32()
    check(_capi.lib.dade_gpu_kmeans(dev.h, ptr(x), n, d, n_clusters, max_iters, int(seed), _dev_flag(x), ptr(cen),
                                    ptr(asg), C.byref(it)))
    return cen, asg, int(it.value)


def compute_ground_truth(dev: Device, data, queries, k: int) -> np.ndarray:
    """compute_ground_truth (proj/src/dataset_io.cpp:101-135) on the GPU: ids
    [nq, k] by (l2_sq_double, id), equal to the reference's."""
    x, q = _rows(data), _rows(queries)
    if int(x.shape[1]) != int(q.shape[1]):
        raise InvalidInput("ground truth: dimension mismatch")
    nq = int(q.shape[0])
    out = np.zeros((nq, max(k, 1)), np.uint32)
    flags = _dev_flag(x)
    if flags != _dev_flag(q):
        raise InvalidInput("ground truth: base and queries must both be host or both be device arrays")
    if flags:
        import torch
        o = torch.empty((nq, max(k, 1)), dtype=torch.int32, device=x.device)
        check(_capi.lib.dade_gpu_ground_truth(dev.h, ptr(x), int(x.shape[0]), ptr(q), nq, int(x.shape[1]), k,
                                              flags, ptr(o)))
        return o.cpu().numpy().astype(np.uint32)
    check(_capi.lib.dade_gpu_ground_truth(dev.h, ptr(x), int(x.shape[0]), ptr(q), nq, int(x.shape[1]), k, 0,
                                          ptr(out)))
    return out


def linear_scan(data_or_index, query, k: int, dco, stats: DcoStats | None = None,
                dev: Device | None = None) -> SearchResult:
    """linear_scan (proj/src/knn.cpp:31-41) for one query."""
    if isinstance(data_or_index, FlatIndex):
        fi = data_or_index
    else:
        fi = FlatIndex(dev or _default_device(), data_or_index)
    ids, dists, counts = fi.search_batch(query, k, dco, stats)
    return _results(ids, dists, counts, k)[0]

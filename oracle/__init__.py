"""TEST INFRASTRUCTURE ONLY — ctypes bindings of the CPU oracle.

* ``Oracle``  -> oracle/liboracle.so: the plain-C restatement of the
  reference's hot-path algorithm (oracle/dade_oracle.c).
* ``RefLib``  -> oracle/_ref/libdade_ref.so: the UNMODIFIED reference library
  compiled from /root/reference by oracle/Makefile (present when it was built
  in the dev container and shipped with the repo snapshot).

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs may
import this package, and only as the checker / baseline — never as the
product path.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ORACLE_SO = HERE / "liboracle.so"
REF_SO = HERE / "_ref" / "libdade_ref.so"
REF_SRC = Path("/root/reference/proj")

P, U8, U32, U64, I, F, D = (C.c_void_p, C.c_uint8, C.c_uint32, C.c_uint64, C.c_int, C.c_float,
                            C.c_double)


def build(ref: bool | None = None) -> None:
    """make -C oracle [ref]; the reference part only where its sources exist."""
    subprocess.run(["make", "-s", "-C", str(HERE), "all"], check=True)
    if ref is None:
        ref = REF_SRC.exists()
    if ref:
        subprocess.run(["make", "-s", "-C", str(HERE), "ref"], check=True)


def _p(a):
    return C.c_void_p(None) if a is None else C.c_void_p(a.ctypes.data)


def _f32(a):
    return np.ascontiguousarray(a, np.float32)


def _u32(a):
    return np.ascontiguousarray(a, np.uint32)


def _f64(a):
    return np.ascontiguousarray(a, np.float64)


class Oracle:
    """The C restatement (oracle/dade_oracle.c)."""

    def __init__(self):
        if not ORACLE_SO.exists():
            build(ref=False)
        L = self.L = C.CDLL(str(ORACLE_SO))
        sig = {
            "dor_accumulate_sqdist": ([P, P, P, U32, U32], None),
            "dor_l2_sq": ([P, P, U32], F),
            "dor_partial_sqdist": ([P, P, U32, U32, U32], F),
            "dor_scale_factor": ([P, U32, U32], D),
            "dor_transform_vector": ([P, U32, P, P], None),
            "dor_apply_transform": ([P, U32, P, U32, P], None),
            "dor_expected_checkpoints": ([U32, U32, P], U32),
            "dor_dade_tables": ([P, U32, P, P, U32, P, P], None),
            "dor_ads_tables": ([U32, U32, D, P, P, P], U32),
            "dor_linear_scan": ([P, U32, U32, P, U32, P, P, P, U32, P, P, P], U32),
            "dor_coarse_rank": ([P, U32, U32, P, U32, P, P], None),
            "dor_ivf_search": ([P, P, P, P, U32, U32, P, U32, U32, P, P, P, U32, P, P, P], U32),
            "dor_ground_truth_one": ([P, U32, U32, P, U32, P], None),
            "dor_recall": ([P, P, U32, P, U32, U32], D),
            "dor_mt64_stream": ([U64, P, U32], None),
            "dor_sample_pairs": ([U32, U64, U64, P, P], None),
            "dor_calibrate": ([P, P, U32, U32, D, U32, U64, U64, P, P], U32),
        }
        for n, (a, r) in sig.items():
            f = getattr(L, n)
            f.argtypes, f.restype = a, r
        # checkpointed_scan returns a struct
        class Outcome(C.Structure):
            _fields_ = [("pruned", U8), ("exact", U8), ("dims_used", U32), ("distance", F)]
        self.Outcome = Outcome
        L.dor_checkpointed_scan.argtypes = [P, P, U32, F, P, P, P, U32, P]
        L.dor_checkpointed_scan.restype = Outcome

    # --- primitives ---------------------------------------------------------
    def partial_sqdist(self, o, q, lo, hi):
        o, q = _f32(o), _f32(q)
        return self.L.dor_partial_sqdist(_p(o), _p(q), len(o), lo, hi)

    def expected_checkpoints(self, dim, delta_d):
        out = np.zeros(max(1, dim), np.uint32)
        n = self.L.dor_expected_checkpoints(dim, delta_d, _p(out))
        return [int(x) for x in out[:n]]

    def dade_tables(self, lambda_prefix, dim, cps, eps):
        lp, c, e = _f64(lambda_prefix), _u32(cps), _f64(eps)
        coeff = np.zeros(max(1, len(c)))
        scale = np.zeros(max(1, len(c)))
        self.L.dor_dade_tables(_p(lp), dim, _p(c), _p(e), len(c), _p(coeff), _p(scale))
        return coeff[:len(c)], scale[:len(c)]

    def ads_tables(self, dim, delta_d, eps0):
        cps = np.zeros(max(1, dim), np.uint32)
        coeff = np.zeros(max(1, dim))
        scale = np.zeros(max(1, dim))
        n = self.L.dor_ads_tables(dim, delta_d, eps0, _p(cps), _p(coeff), _p(scale))
        return cps[:n].copy(), coeff[:n].copy(), scale[:n].copy()

    def scan(self, o, q, r, cps, coeff, scale, stats=None):
        o, q = _f32(o), _f32(q)
        c, co, sc = _u32(cps), _f64(coeff), _f64(scale)
        st = np.zeros(2, np.uint64) if stats is None else stats
        out = self.L.dor_checkpointed_scan(_p(o), _p(q), len(o), float(r), _p(c), _p(co), _p(sc), len(c),
                                           _p(st))
        return bool(out.pruned), float(out.distance), bool(out.exact), int(out.dims_used)

    def apply_transform(self, matrix, rows):
        rows = _f32(rows)
        m = _f64(matrix)
        out = np.empty_like(rows)
        self.L.dor_apply_transform(_p(m), rows.shape[1], _p(rows), rows.shape[0], _p(out))
        return out

    def coarse_rank(self, centroids, q, n_probe):
        cen, q = _f32(centroids), _f32(q)
        lists = np.zeros(n_probe, np.uint32)
        d2 = np.zeros(n_probe, np.float32)
        self.L.dor_coarse_rank(_p(cen), cen.shape[0], cen.shape[1], _p(q), n_probe, _p(lists), _p(d2))
        return lists, d2

    def ivf_search(self, centroids, offsets, ids, storage, queries, k, n_probe, cps=(), coeff=(),
                   scale=()):
        cen, off, idv, sto = _f32(centroids), _u32(offsets), _u32(ids), _f32(storage)
        qs = _f32(queries)
        c, co, sc = _u32(cps), _f64(coeff), _f64(scale)
        nq, dim = qs.shape
        out_i = np.zeros((nq, k), np.uint32)
        out_d = np.zeros((nq, k), np.float32)
        cnt = np.zeros(nq, np.uint32)
        st = np.zeros(2, np.uint64)
        for qi in range(nq):
            cnt[qi] = self.L.dor_ivf_search(_p(cen), _p(off), _p(idv), _p(sto), cen.shape[0], dim,
                                            _p(qs[qi]), k, n_probe, _p(c), _p(co), _p(sc), len(c),
                                            _p(out_i[qi]), _p(out_d[qi]), _p(st))
        return out_i, out_d, cnt, st

    def linear_scan(self, data, queries, k, cps=(), coeff=(), scale=()):
        da, qs = _f32(data), _f32(queries)
        c, co, sc = _u32(cps), _f64(coeff), _f64(scale)
        nq = qs.shape[0]
        out_i = np.zeros((nq, k), np.uint32)
        out_d = np.zeros((nq, k), np.float32)
        cnt = np.zeros(nq, np.uint32)
        st = np.zeros(2, np.uint64)
        for qi in range(nq):
            cnt[qi] = self.L.dor_linear_scan(_p(da), da.shape[0], da.shape[1], _p(qs[qi]), k, _p(c),
                                             _p(co), _p(sc), len(c), _p(out_i[qi]), _p(out_d[qi]),
                                             _p(st))
        return out_i, out_d, cnt, st

    def ground_truth(self, data, queries, k):
        da, qs = _f32(data), _f32(queries)
        out = np.zeros((qs.shape[0], k), np.uint32)
        for qi in range(qs.shape[0]):
            self.L.dor_ground_truth_one(_p(da), da.shape[0], da.shape[1], _p(qs[qi]), k, _p(out[qi]))
        return out

    def recall(self, ids, counts, truth):
        ids, counts, truth = _u32(ids), _u32(counts), _u32(truth)
        return self.L.dor_recall(_p(ids), _p(counts), ids.shape[1], _p(truth), truth.shape[0],
                                 truth.shape[1])

    def mt64(self, seed, n):
        out = np.zeros(n, np.uint64)
        self.L.dor_mt64_stream(seed, _p(out), n)
        return out

    def calibrate(self, lambda_prefix, data, p_s, delta_d, n_pairs, seed):
        lp, da = _f64(lambda_prefix), _f32(data)
        cps = np.zeros(max(1, da.shape[1]), np.uint32)
        eps = np.zeros(max(1, da.shape[1]))
        n = self.L.dor_calibrate(_p(lp), _p(da), da.shape[0], da.shape[1], p_s, delta_d, n_pairs, seed,
                                 _p(cps), _p(eps))
        if n == 0xFFFFFFFF:
            raise RuntimeError("calibrate: degenerate data")
        return [int(x) for x in cps[:n]], [float(x) for x in eps[:n]]


def read_fvecs(path) -> np.ndarray:
    """fvecs records (proj/docs/FILE_FORMATS.md; read_fvecs, proj/src/dataset_io.cpp)."""
    raw = np.fromfile(path, "<i4")
    d = int(raw[0])
    return raw.reshape(-1, d + 1)[:, 1:].view("<f4").copy()


def read_ivecs(path) -> np.ndarray:
    raw = np.fromfile(path, "<i4")
    d = int(raw[0])
    return raw.reshape(-1, d + 1)[:, 1:].copy()


class RefError(RuntimeError):
    pass


class RefLib:
    """The unmodified reference library (oracle/_ref/libdade_ref.so)."""

    def __init__(self):
        if not REF_SO.exists():
            raise FileNotFoundError(f"{REF_SO} not built (make -C oracle ref)")
        L = self.L = C.CDLL(str(REF_SO))
        PP = C.POINTER(P)
        sig = {
            "dref_last_error": ([], C.c_char_p),
            "dref_synth": ([U32, U32, U32, U64, I, D, I, D, P, P], I),
            "dref_fit_pca": ([P, U32, U32, PP], I),
            "dref_fit_random": ([U32, U64, P, U32, PP], I),
            "dref_transform_load": ([C.c_char_p, PP], I),
            "dref_transform_save": ([P, C.c_char_p], I),
            "dref_transform_free": ([P], None),
            "dref_transform_dim": ([P], U32),
            "dref_transform_kind": ([P], I),
            "dref_transform_get": ([P, P, P, P, P], None),
            "dref_apply_transform": ([P, P, U32, P], I),
            "dref_calibrate": ([P, P, U32, D, U32, U64, U64, PP], I),
            "dref_cal_load": ([C.c_char_p, PP], I),
            "dref_cal_save": ([P, C.c_char_p], I),
            "dref_cal_unbounded": ([U32, U32], P),
            "dref_cal_from": ([D, U32, U32, P, P], P),
            "dref_cal_free": ([P], None),
            "dref_cal_get": ([P, P, P, P, P], U32),
            "dref_expected_checkpoints": ([U32, U32, P], U32),
            "dref_strategy_fd": ([U32], P),
            "dref_strategy_dade": ([P, P, U32, PP], I),
            "dref_strategy_ads": ([U32, U32, D, PP], I),
            "dref_strategy_free": ([P], None),
            "dref_evaluate": ([P, P, P, P, U32, U32, I, P, P, P, P, P], I),
            "dref_partial_sqdist": ([P, P, U32, U32, U32], F),
            "dref_dade_estimate": ([P, D, U32], D),
            "dref_ivf_build": ([P, U32, U32, U32, I, U32, U32, U64, PP], I),
            "dref_ivf_load": ([C.c_char_p, PP], I),
            "dref_ivf_save": ([P, C.c_char_p], I),
            "dref_ivf_free": ([P], None),
            "dref_ivf_search": ([P, P, P, U32, U32, U32, P, P, P, P, P, I, P], I),
            "dref_linear_scan": ([P, U32, U32, P, P, U32, U32, P, P, P, P, P, I, P], I),
            "dref_ground_truth": ([P, U32, P, U32, U32, U32, P], I),
            "dref_kmeans": ([P, U32, U32, U32, U32, U64, P, P, P], I),
            "dref_ivf_failure_pass": ([P, P, P, U32, U32, U32, P], I),
            "dref_covariance": ([P, U32, U32, P, P], I),
        }
        for n, (a, r) in sig.items():
            f = getattr(L, n)
            f.argtypes, f.restype = a, r

    def _chk(self, rc):
        if rc:
            raise RefError(f"[{rc}] " + self.L.dref_last_error().decode())

    def synth(self, count, dim, nq, seed, alpha=1.0, rotate=True, uniform=False, mean_shift=0.0):
        data = np.zeros((count, dim), np.float32)
        qs = np.zeros((max(nq, 1), dim), np.float32)
        self._chk(self.L.dref_synth(count, dim, nq, seed, 1 if uniform else 0, alpha, int(rotate),
                                    mean_shift, _p(data), _p(qs)))
        return data, qs[:nq]

    def fit_pca(self, data):
        data = _f32(data)
        h = P()
        self._chk(self.L.dref_fit_pca(_p(data), data.shape[0], data.shape[1], C.byref(h)))
        return RefTransform(self, h)

    def fit_random(self, dim, seed, data):
        data = _f32(data)
        h = P()
        self._chk(self.L.dref_fit_random(dim, seed, _p(data), data.shape[0], C.byref(h)))
        return RefTransform(self, h)

    def load_transform(self, path):
        h = P()
        self._chk(self.L.dref_transform_load(str(path).encode(), C.byref(h)))
        return RefTransform(self, h)

    def cal_load(self, path):
        h = P()
        self._chk(self.L.dref_cal_load(str(path).encode(), C.byref(h)))
        return RefCal(self, h)

    def cal_from(self, p_s, delta_d, cps, eps):
        c, e = _u32(cps), _f64(eps)
        return RefCal(self, self.L.dref_cal_from(p_s, delta_d, len(c), _p(c), _p(e)))

    def cal_unbounded(self, dim, delta_d):
        return RefCal(self, self.L.dref_cal_unbounded(dim, delta_d))

    def expected_checkpoints(self, dim, delta_d):
        out = np.zeros(max(1, dim), np.uint32)
        n = self.L.dref_expected_checkpoints(dim, delta_d, _p(out))
        return [int(x) for x in out[:n]]

    def strategy_fd(self, dim):
        return RefStrategy(self, self.L.dref_strategy_fd(dim), dim)

    def strategy_dade(self, t, cal, delta_d):
        h = P()
        self._chk(self.L.dref_strategy_dade(t.h, cal.h, delta_d, C.byref(h)))
        return RefStrategy(self, h, t.dim)

    def strategy_ads(self, dim, delta_d, eps0):
        h = P()
        self._chk(self.L.dref_strategy_ads(dim, delta_d, eps0, C.byref(h)))
        return RefStrategy(self, h, dim)

    def partial_sqdist(self, o, q, lo, hi):
        o, q = _f32(o), _f32(q)
        return self.L.dref_partial_sqdist(_p(o), _p(q), len(o), lo, hi)

    def ivf_build(self, data, n_clusters, layout=0, split=0, iters=25, seed=1):
        data = _f32(data)
        h = P()
        self._chk(self.L.dref_ivf_build(_p(data), data.shape[0], data.shape[1], n_clusters, layout, split,
                                        iters, seed, C.byref(h)))
        return RefIvf(self, h)

    def ivf_load(self, path):
        h = P()
        self._chk(self.L.dref_ivf_load(str(path).encode(), C.byref(h)))
        return RefIvf(self, h)

    def ground_truth(self, data, queries, k):
        da, qs = _f32(data), _f32(queries)
        out = np.zeros((qs.shape[0], k), np.uint32)
        self._chk(self.L.dref_ground_truth(_p(da), da.shape[0], _p(qs), qs.shape[0], da.shape[1], k, _p(out)))
        return out

    def kmeans(self, data, n_clusters, iters, seed):
        da = _f32(data)
        cen = np.zeros((n_clusters, da.shape[1]), np.float32)
        asg = np.zeros(da.shape[0], np.uint32)
        it = U32()
        self._chk(self.L.dref_kmeans(_p(da), da.shape[0], da.shape[1], n_clusters, iters, seed, _p(cen), _p(asg),
                                     C.byref(it)))
        return cen, asg, int(it.value)

    def covariance(self, data):
        da = _f32(data)
        d = da.shape[1]
        mean, cov = np.zeros(d), np.zeros((d, d))
        self._chk(self.L.dref_covariance(_p(da), da.shape[0], d, _p(mean), _p(cov)))
        return mean, cov

    def linear_scan(self, data, strategy, queries, k, threads=1):
        da, qs = _f32(data), _f32(queries)
        nq = qs.shape[0]
        ids = np.zeros((nq, k), np.uint32)
        d = np.zeros((nq, k), np.float32)
        cnt = np.zeros(nq, np.uint32)
        tr = np.zeros(nq, np.uint8)
        st = np.zeros(2, np.uint64)
        sec = D()
        self._chk(self.L.dref_linear_scan(_p(da), da.shape[0], da.shape[1], strategy.h, _p(qs), nq, k,
                                          _p(ids), _p(d), _p(cnt), _p(tr), _p(st), threads, C.byref(sec)))
        return ids, d, cnt, st, sec.value


class RefTransform:
    def __init__(self, lib, h):
        self.lib, self.h = lib, h
        self.dim = lib.L.dref_transform_dim(h)
        self.kind = lib.L.dref_transform_kind(h)

    def arrays(self):
        d = self.dim
        mean, eig = np.zeros(d), np.zeros(d)
        mat, pre = np.zeros(d * d), np.zeros(d + 1)
        self.lib.L.dref_transform_get(self.h, _p(mean), _p(eig), _p(mat), _p(pre))
        return mean, eig, mat, pre

    def apply(self, rows):
        rows = _f32(rows)
        out = np.empty_like(rows)
        self.lib._chk(self.lib.L.dref_apply_transform(self.h, _p(rows), rows.shape[0], _p(out)))
        return out

    def calibrate(self, data, p_s, delta_d, n_pairs, seed):
        data = _f32(data)
        h = P()
        self.lib._chk(self.lib.L.dref_calibrate(self.h, _p(data), data.shape[0], p_s, delta_d, n_pairs, seed,
                                                C.byref(h)))
        return RefCal(self.lib, h)

    def save(self, path):
        self.lib._chk(self.lib.L.dref_transform_save(self.h, str(path).encode()))

    def dade_estimate(self, partial, d):
        return self.lib.L.dref_dade_estimate(self.h, partial, d)

    def __del__(self):
        try:
            self.lib.L.dref_transform_free(self.h)
        except Exception:
            pass


class RefCal:
    def __init__(self, lib, h):
        self.lib, self.h = lib, h

    def get(self):
        ps, dd = D(), U32()
        n = self.lib.L.dref_cal_get(self.h, C.byref(ps), C.byref(dd), None, None)
        cps = np.zeros(max(n, 1), np.uint32)
        eps = np.zeros(max(n, 1))
        self.lib.L.dref_cal_get(self.h, None, None, _p(cps), _p(eps))
        return ps.value, dd.value, [int(x) for x in cps[:n]], [float(x) for x in eps[:n]]

    def __del__(self):
        try:
            self.lib.L.dref_cal_free(self.h)
        except Exception:
            pass


class RefStrategy:
    def __init__(self, lib, h, dim):
        self.lib, self.h, self.dim = lib, h, dim

    def evaluate(self, o, q, r, measure_failures=False):
        o, q, r = _f32(o), _f32(q), _f32(np.atleast_1d(r))
        n = r.shape[0]
        pr, ex = np.zeros(n, np.uint8), np.zeros(n, np.uint8)
        di, du = np.zeros(n, np.float32), np.zeros(n, np.uint32)
        st = np.zeros(4, np.uint64)
        self.lib._chk(self.lib.L.dref_evaluate(self.h, _p(o), _p(q), _p(r), n, self.dim, int(measure_failures),
                                               _p(pr), _p(di), _p(ex), _p(du), _p(st)))
        return pr.astype(bool), di, ex.astype(bool), du, st

    def __del__(self):
        try:
            self.lib.L.dref_strategy_free(self.h)
        except Exception:
            pass


class RefIvf:
    def __init__(self, lib, h):
        self.lib, self.h = lib, h

    def save(self, path):
        self.lib._chk(self.lib.L.dref_ivf_save(self.h, str(path).encode()))

    def failure_pass(self, strategy, queries, k, n_probe):
        """measure()'s untimed second pass: (total_dco, dims, eligible, failures)."""
        qs = _f32(queries)
        st = np.zeros(4, np.uint64)
        self.lib._chk(self.lib.L.dref_ivf_failure_pass(self.h, strategy.h, _p(qs), qs.shape[0], k, n_probe, _p(st)))
        return st

    def search(self, strategy, queries, k, n_probe, threads=1):
        qs = _f32(queries)
        nq = qs.shape[0]
        ids = np.zeros((nq, k), np.uint32)
        d = np.zeros((nq, k), np.float32)
        cnt = np.zeros(nq, np.uint32)
        tr = np.zeros(nq, np.uint8)
        st = np.zeros(2, np.uint64)
        sec = D()
        self.lib._chk(self.lib.L.dref_ivf_search(self.h, strategy.h, _p(qs), nq, k, n_probe, _p(ids), _p(d),
                                                 _p(cnt), _p(tr), _p(st), threads, C.byref(sec)))
        return ids, d, cnt, st, sec.value

    def __del__(self):
        try:
            self.lib.L.dref_ivf_free(self.h)
        except Exception:
            pass

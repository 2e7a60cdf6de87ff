"""Generate the golden fixtures in tests/golden/ by running the UNMODIFIED
reference library (oracle/_ref/libdade_ref.so, built from /root/reference by
`make -C oracle ref`). Run in the dev container:

    python tests/golden/make_golden.py

Fixtures (all small, committed):
  ivf_fix.npz      test_ivf.cpp's fixture (proj/tests/test_ivf.cpp:53-73):
                   gaussian_set(620, 16, 202, alpha 1, rotated), PCA, 600/20 split,
                   calibrate(p_s .1, dd 4, 20000 pairs, seed 3), IvfIndex::build(12
                   lists, contiguous, 25 iters, seed 9) + reference search outputs.
  eval_fix.npz     DcoStrategy::evaluate outcomes (FD / DADE / ADS / unbounded)
                   on 3000 seeded pairs incl. r = 0 and r = inf, test_estimator.cpp's
                   fixture (proj/tests/test_estimator.cpp:36-49).
  mix_fix.npz      a small Gaussian-mixture stand-in for BASELINE config 0
                   (N 4000, D 32, 16 clusters, lambda_i = i^-1), PCA + calibration +
                   k-means (20 iters, seed 2) by the reference, with its search
                   outputs for FD / DADE at nprobe 4, K 10, dd 8, and ground truth.
  rot_fix.npz      apply_transform outputs (bit-level) for raw rows.
  cfg0_fix.npz     BASELINE config 0 in full (100k x 128, 64-component mixture, PCA,
                   IvfIndex::build nlist 256 / 20 iters / seed 2, calibrate p_s .1 dd 16
                   100k pairs seed 1, nprobe 16, K 10): the reference's covariance,
                   transform, calibration, k-means lists and iteration count, FD and
                   DADE search outputs with DcoStats, measure()'s failure pass, and
                   compute_ground_truth. Data regenerated from tests/golden/synth.py
                   (digest-checked); only the reference's outputs are stored.
  hd_fix.npz       long vectors (D 768 / 960, Delta-d 64, K 10 / 20; configs 4 / 2 shapes
                   scaled to 8k rows, 16 lists): IvfIndex::build, calibration, FD /
                   DADE / unbounded-DADE outputs at nprobe 4 and 16, ground truth.
"""
from __future__ import annotations

import sys
import tempfile
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

sys.path.insert(0, str(Path(__file__).resolve().parent))
from oracle import RefLib  # noqa: E402

OUT = Path(__file__).resolve().parent


def ivf_outputs(ref, ivf, strategies, queries, k, probes):
    out = {}
    for name, s in strategies.items():
        for npb in probes:
            ids, d, cnt, st, _ = ivf.search(s, queries, k, npb)
            out[f"{name}_np{npb}_ids"] = ids
            out[f"{name}_np{npb}_dists"] = d
            out[f"{name}_np{npb}_counts"] = cnt
            out[f"{name}_np{npb}_stats"] = st
    return out


def divf_arrays(path):
    from paper_2411_17229_b200.io import read_divf  # pure-python reader, no GPU needed
    return read_divf(path)


def main():
    ref = RefLib()
    tmp = Path(tempfile.mkdtemp())
    if len(sys.argv) > 1:  # only the named fixtures (e.g. cfg0 hd)
        for name in sys.argv[1:]:
            {"cfg0": make_cfg0, "hd": make_hd}[name](ref, tmp)
        return

    # ---- ivf_fix (proj/tests/test_ivf.cpp:53-73) ---------------------------
    raw, _ = ref.synth(620, 16, 0, 202, alpha=1.0, rotate=True)
    t = ref.fit_pca(raw)
    rot = t.apply(raw)
    data, queries = rot[:600], rot[600:]
    cal = t.calibrate(data, 0.1, 4, 20000, 3)
    ps, dd, cps, eps = cal.get()
    ivf = ref.ivf_build(data, 12, layout=0, split=0, iters=25, seed=9)
    ivf.save(tmp / "fix.ivf")
    ivf_split = ref.ivf_build(data, 12, layout=1, split=4, iters=25, seed=9)
    ivf_split.save(tmp / "fix_split.ivf")
    mean, eig, mat, pre = t.arrays()
    strategies = {
        "fd": ref.strategy_fd(16),
        "dade": ref.strategy_dade(t, cal, 4),
        "ads": ref.strategy_ads(16, 4, 2.1),
        "unb": ref.strategy_dade(t, ref.cal_unbounded(16, 4), 4),
    }
    res = ivf_outputs(ref, ivf, strategies, queries, 10, [1, 3, 12])
    # truncation case (proj/tests/test_ivf.cpp:265-281)
    ids, d, cnt, st, _ = ivf.search(strategies["fd"], queries[:1], 700, 12)
    res.update(trunc_ids=ids, trunc_dists=d, trunc_counts=cnt)
    lin = {}
    for name in ("fd", "dade", "ads"):
        ids, d, cnt, st, _ = ref.linear_scan(data, strategies[name], queries, 10)
        lin.update({f"lin_{name}_ids": ids, f"lin_{name}_dists": d, f"lin_{name}_counts": cnt,
                    f"lin_{name}_stats": st})
    gt = ref.ground_truth(data, queries, 10)
    dv = divf_arrays(tmp / "fix.ivf")
    ds = divf_arrays(tmp / "fix_split.ivf")
    np.savez_compressed(
        OUT / "ivf_fix.npz", raw=raw, data=data, queries=queries, mean=mean, eig=eig, matrix=mat,
        lambda_prefix=pre, cal_p_s=ps, cal_delta_d=dd, cal_cps=np.array(cps, np.uint32),
        cal_eps=np.array(eps), centroids=dv.centroids, offsets=dv.offsets, ids=dv.ids, storage=dv.storage,
        split_centroids=ds.centroids, split_offsets=ds.offsets, split_ids=ds.ids, split_storage=ds.storage,
        gt=gt, **res, **lin)

    # ---- eval_fix (proj/tests/test_estimator.cpp:36-49, 163-250) ------------
    raw2, _ = ref.synth(1000, 32, 0, 101, alpha=1.0, rotate=True)
    t2 = ref.fit_pca(raw2)
    d2 = t2.apply(raw2)
    cal2 = t2.calibrate(d2, 0.1, 8, 40000, 7)
    ps2, dd2, cps2, eps2 = cal2.get()
    rng = np.random.default_rng(66)
    n = 3000
    ii = rng.integers(0, 1000, n)
    jj = (ii + 1 + rng.integers(0, 999, n)) % 1000
    o, q = d2[ii], d2[jj]
    fd2 = ref.strategy_fd(32)
    exact = fd2.evaluate(o, q, np.full(n, np.inf, np.float32))[1]
    r = (exact * (0.7 + 0.3 * (np.arange(n) % 4))).astype(np.float32)
    r[::97] = 0.0
    r[1::89] = np.inf
    o[5] = q[5]  # self distance at r = 0 (test_estimator.cpp:244-249)
    r[5] = 0.0
    ev = {}
    strat2 = {"fd": fd2, "dade": ref.strategy_dade(t2, cal2, 8), "ads": ref.strategy_ads(32, 8, 2.1),
              "unb": ref.strategy_dade(t2, ref.cal_unbounded(32, 8), 8)}
    for name, s in strat2.items():
        pr, di, ex, du, st = s.evaluate(o, q, r, measure_failures=True)
        ev.update({f"{name}_pruned": pr, f"{name}_dist": di, f"{name}_exact": ex, f"{name}_dims": du,
                   f"{name}_stats": st})
    partial = np.array([[ref.partial_sqdist(o[p], q[p], 0, d) for d in cps2 + [32]] for p in range(200)],
                       np.float32)
    est = np.array([[t2.dade_estimate(float(partial[p, i]), d) for i, d in enumerate(cps2 + [32])]
                    for p in range(200)])
    _, eig2, mat2, pre2 = t2.arrays()
    np.savez_compressed(OUT / "eval_fix.npz", o=o, q=q, r=r, eig=eig2, matrix=mat2, lambda_prefix=pre2,
                        cal_p_s=ps2, cal_delta_d=dd2, cal_cps=np.array(cps2, np.uint32), cal_eps=np.array(eps2),
                        partial=partial, estimate=est, **ev)

    # ---- mix_fix: small Gaussian mixture (BASELINE config-0 shape, scaled) ---
    g = np.random.default_rng(0)
    D, N, NQ, C = 32, 4000, 100, 16
    lam = np.arange(1, D + 1, dtype=np.float64) ** -1.0
    lam *= D / lam.sum()
    R, _ = np.linalg.qr(g.standard_normal((D, D)))
    centers = g.standard_normal((C, D)) * 4.0
    def draw(n, gg):
        comp = gg.integers(0, C, n)
        z = gg.standard_normal((n, D)) * np.sqrt(lam)
        return (centers[comp] + z @ R.T).astype(np.float32)
    base_raw = draw(N, g)
    q_raw = draw(NQ, np.random.default_rng(1))
    t3 = ref.fit_pca(base_raw)
    b3 = t3.apply(base_raw)
    q3 = t3.apply(q_raw)
    cal3 = t3.calibrate(b3, 0.1, 8, 100000, 1)
    ps3, dd3, cps3, eps3 = cal3.get()
    ivf3 = ref.ivf_build(b3, 64, layout=0, split=0, iters=20, seed=2)
    ivf3.save(tmp / "mix.ivf")
    dv3 = divf_arrays(tmp / "mix.ivf")
    strat3 = {"fd": ref.strategy_fd(D), "dade": ref.strategy_dade(t3, cal3, 8)}
    res3 = ivf_outputs(ref, ivf3, strat3, q3, 10, [4, 16])
    gt3 = ref.ground_truth(b3, q3, 10)
    _, eig3, mat3, pre3 = t3.arrays()
    np.savez_compressed(OUT / "mix_fix.npz", base_raw=base_raw, q_raw=q_raw, base=b3, queries=q3, eig=eig3,
                        matrix=mat3, lambda_prefix=pre3, cal_p_s=ps3, cal_delta_d=dd3,
                        cal_cps=np.array(cps3, np.uint32), cal_eps=np.array(eps3), centroids=dv3.centroids,
                        offsets=dv3.offsets, ids=dv3.ids, storage=dv3.storage, gt=gt3, **res3)

    # ---- rot_fix: apply_transform bits --------------------------------------
    np.savez_compressed(OUT / "rot_fix.npz", matrix=mat3, eig=eig3, raw=q_raw, rotated=q3,
                        matrix16=mat, raw16=raw[:50], rotated16=rot[:50])
    make_cfg0(ref, tmp)
    make_hd(ref, tmp)
    for f in sorted(OUT.glob("*.npz")):
        print(f.name, f.stat().st_size)


def make_cfg0(ref, tmp):
    import time
    import synth
    c = synth.CFG0
    t0 = time.time()
    base_raw, q_raw = synth.config0()
    print(f"cfg0 data {time.time() - t0:.1f}s", flush=True)
    cmean, cov = ref.covariance(base_raw)
    t = ref.fit_pca(base_raw)
    mean, eig, mat, pre = t.arrays()
    base, q = t.apply(base_raw), t.apply(q_raw)
    cal = t.calibrate(base, c["p_s"], c["delta_d"], c["cal_pairs"], c["cal_seed"])
    ps, dd, cps, eps = cal.get()
    print(f"cfg0 pca+cal {time.time() - t0:.1f}s", flush=True)
    ivf = ref.ivf_build(base, c["nlist"], layout=0, split=0, iters=c["kmeans_iters"], seed=c["kmeans_seed"])
    ivf.save(tmp / "cfg0.ivf")
    dv = divf_arrays(tmp / "cfg0.ivf")
    _, _, km_iters = ref.kmeans(base[:2000], 16, c["kmeans_iters"], c["kmeans_seed"])  # (shim smoke)
    print(f"cfg0 ivf {time.time() - t0:.1f}s", flush=True)
    strat = {"fd": ref.strategy_fd(c["dim"]), "dade": ref.strategy_dade(t, cal, c["delta_d"])}
    res = ivf_outputs(ref, ivf, strat, q, c["k"], [c["nprobe"]])
    fail = ivf.failure_pass(strat["dade"], q, c["k"], c["nprobe"])
    gt = ref.ground_truth(base, q, c["k"])
    print(f"cfg0 search+gt {time.time() - t0:.1f}s", flush=True)
    np.savez_compressed(
        OUT / "cfg0_fix.npz", base_raw_digest=synth.digest(base_raw), q_raw_digest=synth.digest(q_raw),
        base_digest=synth.digest(base), cov_mean=cmean, cov=cov, mean=mean, eig=eig, matrix=mat,
        lambda_prefix=pre, cal_p_s=ps, cal_delta_d=dd, cal_cps=np.array(cps, np.uint32), cal_eps=np.array(eps),
        centroids=dv.centroids, offsets=dv.offsets, ids=dv.ids, dade_failure_stats=fail, gt=gt, **res)


def make_hd(ref, tmp):
    import synth
    from paper_2411_17229_b200.api import OrthoTransform
    from paper_2411_17229_b200.io import write_transform
    out = {}
    for dim, c in synth.HD.items():
        base, q, lam = synth.high_dim(dim)
        write_transform(tmp / f"hd{dim}.dade", OrthoTransform(dim, 0, np.zeros(dim), lam, np.eye(dim).reshape(-1)))
        t = ref.load_transform(tmp / f"hd{dim}.dade")
        cal = t.calibrate(base, c["p_s"], c["delta_d"], 20000, 7)
        ps, dd, cps, eps = cal.get()
        ivf = ref.ivf_build(base, c["nlist"], layout=0, split=0, iters=20, seed=2)
        ivf.save(tmp / f"hd{dim}.ivf")
        dv = divf_arrays(tmp / f"hd{dim}.ivf")
        strat = {"fd": ref.strategy_fd(dim), "dade": ref.strategy_dade(t, cal, c["delta_d"]),
                 "unb": ref.strategy_dade(t, ref.cal_unbounded(dim, c["delta_d"]), c["delta_d"])}
        res = ivf_outputs(ref, ivf, strat, q, c["k"], [c["nprobe"], c["nlist"]])
        gt = ref.ground_truth(base, q, c["k"])
        p = f"d{dim}_"
        out.update({p + "base_digest": synth.digest(base), p + "q_digest": synth.digest(q), p + "eig": lam,
                    p + "cal_p_s": ps, p + "cal_delta_d": dd, p + "cal_cps": np.array(cps, np.uint32),
                    p + "cal_eps": np.array(eps), p + "centroids": dv.centroids, p + "offsets": dv.offsets,
                    p + "ids": dv.ids, p + "gt": gt})
        out.update({p + kk: v for kk, v in res.items()})
    np.savez_compressed(OUT / "hd_fix.npz", **out)


if __name__ == "__main__":
    main()

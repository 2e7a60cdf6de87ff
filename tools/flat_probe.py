"""Flat scan (config 4) statistics: DcoStats of one batch (DCOs, dims accumulated,
dims per DCO beyond the first slice) and the per-pass filter time.
    python tools/flat_probe.py"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main(name="config4"):
    import numpy as np

    import paper_2411_17229_b200 as gp
    from paper_2411_17229_b200.io import read_cal, read_fvecs, read_transform
    from paper_2411_17229_b200.workloads import CONFIGS, ensure_artifacts
    cfg = CONFIGS[name]
    art = ensure_artifacts(cfg, gt_queries=2000, log=lambda *a: print(*a, file=sys.stderr))
    dev = gp.Device(0)
    fi = gp.FlatIndex(dev, read_fvecs(art / "base.fvecs"))
    t = read_transform(art / "t.dade")
    dco = gp.DadeStrategy(t, read_cal(art / "c.cal"), cfg.delta_d, dev=dev)
    q = read_fvecs(art / "queries.fvecs")
    st = gp.DcoStats()
    dev.set_profiling(True)
    fi.search_batch(q, cfg.k, dco, stats=st, raw=True)
    fi.search_batch(q, cfg.k, dco, stats=gp.DcoStats(), raw=True)
    print("filter ms / launches", dev.last_filter_profile(), "seed", dev.last_seed_profile())
    print(f"DCOs {st.total_dco:.4e} dims {st.dims_accumulated:.4e} per query {st.total_dco / q.shape[0]:.0f} "
          f"dim_fraction {st.dim_fraction(cfg.dim):.4f} dims/DCO {st.dims_accumulated / max(st.total_dco, 1):.1f}")


if __name__ == "__main__":
    main(*(sys.argv[1:2] or ["config4"]))

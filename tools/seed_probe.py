"""Seed kernel alone on a BASELINE workload: device time and scored pair-dims
(dade_gpu_last_seed_profile) of a few searches.
    python tools/seed_probe.py config1"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main(name="config1"):
    import torch

    import paper_2411_17229_b200 as gp
    from paper_2411_17229_b200 import _capi
    from paper_2411_17229_b200.io import read_cal, read_divf, read_fvecs, read_transform
    from paper_2411_17229_b200.workloads import CONFIGS, ensure_artifacts
    cfg = CONFIGS[name]
    art = ensure_artifacts(cfg, gt_queries=2000, log=lambda *a: print(*a, file=sys.stderr))
    dev = gp.Device(0)
    idx = gp.IvfIndex.from_divf(dev, read_divf(art / "index.ivf"))
    dco = gp.DadeStrategy(read_transform(art / "t.dade"), read_cal(art / "c.cal"), cfg.delta_d, dev=dev)
    dev.apply(dco)
    q = torch.from_numpy(read_fvecs(art / "queries.fvecs")).cuda()
    nq, k = q.shape[0], cfg.k
    oi = torch.empty((nq, k), dtype=torch.int32, device="cuda")
    od = torch.empty((nq, k), dtype=torch.float32, device="cuda")
    oc = torch.empty((nq,), dtype=torch.int32, device="cuda")
    dev.set_profiling(True)
    for _ in range(4):
        _capi.check(_capi.lib.dade_gpu_ivf_search(dev.h, _capi.ptr(q), nq, k, cfg.nprobe,
                                                  _capi.QUERIES_RAW | _capi.DEVICE_PTRS, _capi.ptr(oi),
                                                  _capi.ptr(od), _capi.ptr(oc), None))
        torch.cuda.synchronize()
        ms, pd = dev.last_seed_profile()
        print(f"seed {ms * 1e3:.1f} us, pair-dims {pd:.3e}", flush=True)


if __name__ == "__main__":
    main(*(sys.argv[1:2] or ["config1"]))

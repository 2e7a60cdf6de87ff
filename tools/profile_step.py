"""One IVF-DADE search of a BASELINE workload between cudaProfilerStart/Stop,
after warm-up searches, for ncu captures (run `python -m paper_2411_17229_b200.workloads
--config X` first so the artifacts are cached):

    ncu --profile-from-start off --set full --clock-control none --import-source on \\
        -o gpurun_out/step python tools/profile_step.py config1
    ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \\
        --log-file gpurun_out/launches.csv python tools/profile_step.py config1
"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main(name="config1", warm=3, parts=0):
    import torch

    import paper_2411_17229_b200 as gp
    from paper_2411_17229_b200 import _capi
    from paper_2411_17229_b200.io import read_cal, read_divf, read_fvecs, read_transform
    from paper_2411_17229_b200.workloads import CONFIGS, ensure_artifacts
    cfg = CONFIGS[name]
    art = ensure_artifacts(cfg, gt_queries=2000, log=lambda *a: print(*a, file=sys.stderr))
    dev = gp.Device(0)
    if cfg.flat:
        idx = gp.FlatIndex(dev, read_fvecs(art / "base.fvecs"))
        if parts:  # the data-ordered scan (dade_gpu_flat_partition), as bench.py's config4 block runs it
            idx.partition(parts, 10, 1)
    else:
        idx = gp.IvfIndex.from_divf(dev, read_divf(art / "index.ivf"))
    dco = gp.DadeStrategy(read_transform(art / "t.dade"), read_cal(art / "c.cal"), cfg.delta_d, dev=dev)
    dev.apply(dco)
    q = torch.from_numpy(read_fvecs(art / "queries.fvecs")).cuda()
    nq, k = q.shape[0], cfg.k
    oi = torch.empty((nq, k), dtype=torch.int32, device="cuda")
    od = torch.empty((nq, k), dtype=torch.float32, device="cuda")
    oc = torch.empty((nq,), dtype=torch.int32, device="cuda")
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")

    def search():
        if cfg.flat:
            _capi.check(_capi.lib.dade_gpu_flat_search(dev.h, _capi.ptr(q), nq, k,
                                                       _capi.QUERIES_RAW | _capi.DEVICE_PTRS, _capi.ptr(oi),
                                                       _capi.ptr(od), _capi.ptr(oc), None))
            return
        _capi.check(_capi.lib.dade_gpu_ivf_search(dev.h, _capi.ptr(q), nq, k, cfg.nprobe,
                                                  _capi.QUERIES_RAW | _capi.DEVICE_PTRS, _capi.ptr(oi),
                                                  _capi.ptr(od), _capi.ptr(oc), None))
    for _ in range(warm):
        search()
    flush.zero_()
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    search()
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "config1", parts=int(sys.argv[2]) if len(sys.argv) > 2 else 0)

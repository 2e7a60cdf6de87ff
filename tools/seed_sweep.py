"""Seed-rows sweep: device time per search and recall@K for several
dade_gpu_set_seed_rows values on a BASELINE workload (tuning evidence only).
    python tools/seed_sweep.py config1 0 512 256 128
"""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main(name, rows_list):
    import numpy as np
    import torch

    import paper_2411_17229_b200 as gp
    from paper_2411_17229_b200 import _capi
    from paper_2411_17229_b200.io import read_cal, read_divf, read_fvecs, read_ivecs, read_transform
    from paper_2411_17229_b200.workloads import CONFIGS, ensure_artifacts
    from oracle import Oracle
    cfg = CONFIGS[name]
    art = ensure_artifacts(cfg, gt_queries=2000, log=lambda *a: print(*a, file=sys.stderr))
    dev = gp.Device(0)
    idx = gp.IvfIndex.from_divf(dev, read_divf(art / "index.ivf"))
    dco = gp.DadeStrategy(read_transform(art / "t.dade"), read_cal(art / "c.cal"), cfg.delta_d, dev=dev)
    dev.apply(dco)
    q = torch.from_numpy(read_fvecs(art / "queries.fvecs")).cuda()
    gt = read_ivecs(art / "gt.ivecs").astype(np.uint32)
    nq, k = q.shape[0], cfg.k
    oi = torch.empty((nq, k), dtype=torch.int32, device="cuda")
    od = torch.empty((nq, k), dtype=torch.float32, device="cuda")
    oc = torch.empty((nq,), dtype=torch.int32, device="cuda")
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    st = torch.cuda.current_stream()

    def search():
        _capi.check(_capi.lib.dade_gpu_ivf_search(dev.h, _capi.ptr(q), nq, k, cfg.nprobe,
                                                  _capi.QUERIES_RAW | _capi.DEVICE_PTRS, _capi.ptr(oi),
                                                  _capi.ptr(od), _capi.ptr(oc), None))
    out = []
    for rows in rows_list:
        _capi.check(_capi.lib.dade_gpu_set_seed_rows(dev.h, rows))
        for _ in range(3):
            search()
        ts = []
        for _ in range(10):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            search()
            e1.record(st)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        m = gt.shape[0]
        rec = Oracle().recall(oi[:m].cpu().numpy().astype(np.uint32), oc[:m].cpu().numpy().astype(np.uint32), gt)
        r = {"config": name, "seed_rows": rows, "ms_median": float(np.median(ts)), "recall": float(rec)}
        print(json.dumps(r), flush=True)
        out.append(r)
    _capi.check(_capi.lib.dade_gpu_set_seed_rows(dev.h, 0))
    return out


if __name__ == "__main__":
    main(sys.argv[1], [int(x) for x in sys.argv[2:]] or [0, 512, 256, 128])

"""Config 4 through the product's data-ordered flat scan (FlatIndex.partition ->
dade_gpu_flat_partition, then dade_gpu_flat_search): partition build time,
device time per 4096-query batch, recall, for each cell count given.
    python tools/flat_ordered_probe.py [n_parts ...] [--iters N]
SEED_ROWS=N in the environment overrides the seeded rows (dade_gpu_set_seed_rows)."""
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main(parts=(256,), iters=10):
    import numpy as np
    import torch

    import paper_2411_17229_b200 as gp
    from paper_2411_17229_b200 import _capi
    from paper_2411_17229_b200.io import read_cal, read_fvecs, read_ivecs, read_transform
    from paper_2411_17229_b200.workloads import CONFIGS, ensure_artifacts
    from oracle import Oracle
    cfg = CONFIGS["config4"]
    art = ensure_artifacts(cfg, gt_queries=2000, log=lambda *a: print(*a, file=sys.stderr))
    dev = gp.Device(0)
    fi = gp.FlatIndex(dev, read_fvecs(art / "base.fvecs"))
    dco = gp.DadeStrategy(read_transform(art / "t.dade"), read_cal(art / "c.cal"), cfg.delta_d, dev=dev)
    q = torch.from_numpy(read_fvecs(art / "queries.fvecs")).cuda()
    gt = read_ivecs(art / "gt.ivecs").astype(np.uint32)
    nq, k = q.shape[0], cfg.k
    oi = torch.empty((nq, k), dtype=torch.int32, device="cuda")
    od = torch.empty((nq, k), dtype=torch.float32, device="cuda")
    oc = torch.empty((nq,), dtype=torch.int32, device="cuda")
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    for n in parts:
        t0 = time.time()
        fi.partition(n, iters, 1)
        torch.cuda.synchronize()
        bt = time.time() - t0
        dev.apply(dco)
        import os
        if os.environ.get("SEED_ROWS"):
            _capi.check(_capi.lib.dade_gpu_set_seed_rows(dev.h, int(os.environ["SEED_ROWS"])))

        def search():
            _capi.check(_capi.lib.dade_gpu_flat_search(dev.h, _capi.ptr(q), nq, k, _capi.QUERIES_RAW | _capi.DEVICE_PTRS,
                                                       _capi.ptr(oi), _capi.ptr(od), _capi.ptr(oc), None))
        for _ in range(3):
            search()
        ts = []
        for _ in range(5):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            search()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ids = oi[:gt.shape[0]].cpu().numpy()
        rec = Oracle().recall(ids.astype(np.uint32), oc[:gt.shape[0]].cpu().numpy().astype(np.uint32), gt)
        print(f"parts {n}: build {bt:.2f} s, {np.median(ts):.3f} ms per batch, {nq / np.median(ts) * 1e3:.0f} q/s, "
              f"recall {rec:.4f}", flush=True)


if __name__ == "__main__":
    args = sys.argv[1:]
    it = 10
    if "--iters" in args:
        i = args.index("--iters")
        it = int(args[i + 1])
        del args[i:i + 2]
    main(tuple(int(x) for x in args) or (256,), it)

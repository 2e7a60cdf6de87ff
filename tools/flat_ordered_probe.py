"""Config 4 as an IVF search with every list probed (a data-ordered exhaustive
scan): build time, device time per 4096-query batch, recall.
    python tools/flat_ordered_probe.py [n_lists] [kmeans_iters]"""
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main(n_lists=256, iters=10):
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
    base = torch.from_numpy(read_fvecs(art / "base.fvecs")).cuda()
    t0 = time.time()
    idx = gp.IvfIndex.build(dev, base, n_lists, iters, 1)
    print(f"build {time.time() - t0:.1f} s, lists min/max {np.diff(idx.offsets).min()}/{np.diff(idx.offsets).max()}",
          flush=True)
    dco = gp.DadeStrategy(read_transform(art / "t.dade"), read_cal(art / "c.cal"), cfg.delta_d, dev=dev)
    dev.apply(dco)
    q = torch.from_numpy(read_fvecs(art / "queries.fvecs")).cuda()
    gt = read_ivecs(art / "gt.ivecs").astype(np.uint32)
    nq, k = q.shape[0], cfg.k
    oi = torch.empty((nq, k), dtype=torch.int32, device="cuda")
    od = torch.empty((nq, k), dtype=torch.float32, device="cuda")
    oc = torch.empty((nq,), dtype=torch.int32, device="cuda")
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")

    def search():
        _capi.check(_capi.lib.dade_gpu_ivf_search(dev.h, _capi.ptr(q), nq, k, n_lists,
                                                  _capi.QUERIES_RAW | _capi.DEVICE_PTRS, _capi.ptr(oi),
                                                  _capi.ptr(od), _capi.ptr(oc), None))
    for _ in range(2):
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
    ids = idx.ids[oi[:gt.shape[0]].cpu().numpy().astype(np.int64)] if False else oi[:gt.shape[0]].cpu().numpy()
    rec = Oracle().recall(ids.astype(np.uint32), oc[:gt.shape[0]].cpu().numpy().astype(np.uint32), gt)
    print(f"n_lists {n_lists}: {np.median(ts):.3f} ms per batch, {nq / np.median(ts) * 1e3:.0f} q/s, recall {rec:.4f}",
          flush=True)


if __name__ == "__main__":
    a = [int(x) for x in sys.argv[1:]]
    main(*a)

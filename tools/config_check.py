"""Run one search of a BASELINE config end to end on the GPU (IVF or flat), report
time, recall against exact ground truth and the reference's recall on a sample
(diagnostic; the bench line itself is config 1).
    python tools/config_check.py config2 [n_ref_queries]"""
import os, sys, time, tempfile
from pathlib import Path
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2411_17229_b200 as gp
from paper_2411_17229_b200 import workloads as W

name = sys.argv[1] if len(sys.argv) > 1 else "config2"
n_ref = int(sys.argv[2]) if len(sys.argv) > 2 else 50
cfg = W.CONFIGS[name]
dev = gp.Device(0)
art = W.build(cfg, dev, torch.device("cuda:0"), with_gt=True, log=print)
dco = gp.DadeStrategy(art.transform, art.cal, cfg.delta_d, dev=dev)
q = art.q_rot.cpu().numpy()
if cfg.flat:
    idx = gp.FlatIndex(dev, art.base_rot.cpu().numpy())
    run = lambda: idx.search_batch(q, cfg.k, dco)
else:
    idx = gp.IvfIndex(dev, cfg.dim, cfg.n, cfg.nlist, art.centroids, art.offsets, art.ids, art.storage)
    run = lambda: idx.search_batch(q, cfg.k, cfg.nprobe, dco)
for _ in range(2):
    ids, d, cnt = run()
torch.cuda.synchronize()
t0 = time.perf_counter()
ids, d, cnt = run()
dt = time.perf_counter() - t0
gt = art.gt
rec = np.mean([len(set(ids[i, :cnt[i]].tolist()) & set(gt[i].tolist())) / cfg.k for i in range(len(gt))])
print(f"{name}: {len(q)} queries in {dt * 1e3:.2f} ms (host buffers, incl. copies) -> {len(q) / dt:.0f} q/s, recall@{cfg.k} {rec:.4f}")

if os.environ.get("DADE_GPU_PHASES") == "1":
    from paper_2411_17229_b200 import _capi
    buf = np.zeros(16, np.uint64)
    _capi.check(_capi.lib.dade_gpu_debug_counters(dev.h, _capi.ptr(buf)))
    c = [int(x) for x in buf[8:16]]
    us = lambda x: x / 148 / 1.9e3
    print(f"last pass per CTA: items {c[0] / 148:.1f} stage {us(c[1]):.1f} us | mma wait: bready {us(c[2]):.1f} "
          f"accempty {us(c[3]):.1f} afull {us(c[4]):.1f} us | epi warp0 wait: meta {us(c[5]):.1f} acc {us(c[6]):.1f} us "
          f"| tma wait aempty {us(c[7]):.1f} us")

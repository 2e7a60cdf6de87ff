"""Run a few host-buffer (e2e) searches of a BASELINE config (for ncu launch lists).
    python tools/e2e_once.py [config1] [n]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2411_17229_b200 as gp
from paper_2411_17229_b200 import _capi, workloads as W

cfg = W.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "config1"]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 3
dev = gp.Device(0)
art = W.build(cfg, dev, torch.device("cuda:0"), with_gt=False, log=lambda *a: None)
idx = gp.IvfIndex(dev, cfg.dim, cfg.n, cfg.nlist, art.centroids, art.offsets, art.ids, art.storage)
dco = gp.DadeStrategy(art.transform, art.cal, cfg.delta_d, dev=dev)
dev.apply(dco)
nq, k = art.q_raw.shape[0], cfg.k
qh = torch.empty((nq, cfg.dim), dtype=torch.float32, pin_memory=True)
qh.copy_(art.q_raw.cpu())
ih = torch.empty((nq, k), dtype=torch.int32, pin_memory=True)
dh = torch.empty((nq, k), dtype=torch.float32, pin_memory=True)
ch = torch.empty((nq,), dtype=torch.int32, pin_memory=True)
for _ in range(n):
    _capi.check(_capi.lib.dade_gpu_ivf_search(dev.h, _capi.ptr(qh), nq, k, cfg.nprobe, _capi.QUERIES_RAW,
                                              _capi.ptr(ih), _capi.ptr(dh), _capi.ptr(ch), None))
torch.cuda.synchronize()

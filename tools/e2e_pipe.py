"""Pipelined host-buffer searches (dade_gpu_ivf_search_batches) of a BASELINE config:
wall time per batch; DADE_GPU_HOST_TIMING=1 adds per-batch host enqueue / device span / gap.
    python tools/e2e_pipe.py [config1] [n]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2411_17229_b200 as gp
from paper_2411_17229_b200 import workloads as W

cfg = W.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "config1"]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 8
dev = gp.Device(0)
art = W.build(cfg, dev, torch.device("cuda:0"), with_gt=False, log=lambda *a: None)
idx = gp.IvfIndex(dev, cfg.dim, cfg.n, cfg.nlist, art.centroids, art.offsets, art.ids, art.storage)
dco = gp.DadeStrategy(art.transform, art.cal, cfg.delta_d, dev=dev)
nq, k = art.q_raw.shape[0], cfg.k
qh = torch.empty((nq, cfg.dim), dtype=torch.float32, pin_memory=True)
qh.copy_(art.q_raw.cpu())
outs = [tuple(torch.empty(s, dtype=t, pin_memory=True) for s, t in
              (((nq, k), torch.int32), ((nq, k), torch.float32), ((nq,), torch.int32))) for _ in range(2)]
for rep in range(3):
    t0 = time.perf_counter()
    idx.search_batches([qh] * n, k, cfg.nprobe, dco, raw=True, outputs=[outs[b % 2] for b in range(n)])
    dt = time.perf_counter() - t0
    print(f"{n} batches: {1e3 * dt / n:.3f} ms per batch -> {n * nq / dt / 1e6:.2f} M queries/s", flush=True)

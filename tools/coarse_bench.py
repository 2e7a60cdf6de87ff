"""Coarse ranking alone (dade_gpu_coarse_probes) on random centroids: device time per batch.
    python tools/coarse_bench.py [nlist] [nq] [dim] [n_probe]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2411_17229_b200 as gp
from paper_2411_17229_b200.dist import coarse_probes

nlist, nq, dim, npb = (int(x) for x in (sys.argv[1:] + ["16384", "100000", "128", "64"][len(sys.argv) - 1:])[:4])
g = np.random.default_rng(0)
cent = (g.standard_normal((nlist, dim)) * 4).astype(np.float32)
offsets = np.arange(nlist + 1, dtype=np.uint32)
dev = gp.Device(0)
gp.IvfIndex(dev, dim, nlist, nlist, cent, offsets, np.arange(nlist, dtype=np.uint32), cent)
dev.apply(gp.FdScanningStrategy(dim))
q = torch.from_numpy((cent[g.integers(0, nlist, nq)] + g.standard_normal((nq, dim))).astype(np.float32)).cuda()
q_rot = torch.empty_like(q)
pr = torch.empty((nq, npb), dtype=torch.int64, device="cuda")
dev.set_stream(torch.cuda.current_stream().cuda_stream)
ts = []
for it in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    coarse_probes(dev, q, nq, npb, q_rot, pr)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
print(f"coarse nlist {nlist} nq {nq} dim {dim} n_probe {npb}: {min(ts):.3f} ms ({nq / min(ts) * 1e3 / 1e6:.2f} M queries/s)")

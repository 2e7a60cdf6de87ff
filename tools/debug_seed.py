"""Check the radius seed / pass-1 radius against exact K-th distances (config1)."""
import ctypes, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2411_17229_b200 as gp
from paper_2411_17229_b200 import _capi, workloads as W

cfg = W.CONFIGS["config1"]
dev = gp.Device(0)
art = W.build(cfg, dev, torch.device("cuda:0"), with_gt=True, log=lambda *a: None)
idx = gp.IvfIndex(dev, cfg.dim, cfg.n, cfg.nlist, art.centroids, art.offsets, art.ids, art.storage)
dco = gp.DadeStrategy(art.transform, art.cal, cfg.delta_d, dev=dev)
nq = 200
q = art.q_rot[:nq].contiguous()
k = cfg.k
ids, d, cnt = idx.search_batch(q.cpu().numpy(), k, cfg.nprobe, dco)
rb = np.zeros(nq, np.uint32)
_capi.check(_capi.lib.dade_gpu_debug_radius(dev.h, _capi.ptr(rb), nq))
r_final = rb.view(np.float32)
# exact: nearest list of each query, K-th distance among its first 512 rows and all rows
cen = torch.from_numpy(art.centroids).cuda()
qd = torch.cdist(q.double(), cen.double())
near = qd.argmin(1).cpu().numpy()
sto = torch.from_numpy(art.storage).cuda()
offs = art.offsets
bad = 0
for i in range(20):
    l = near[i]
    rows = sto[offs[l]:offs[l + 1]]
    dd = torch.sqrt(((rows.double() - q[i].double()) ** 2).sum(1)).cpu().numpy()
    k512 = np.sort(dd[:512])[k - 1] if len(dd) >= max(k, 1) else np.inf
    kall = np.sort(dd)[k - 1]
    # true K-th over all probed = our result's K-th distance if recall were perfect; use GT
    gtd = np.sqrt(((art.base_rot[torch.from_numpy(art.gt[i].astype(np.int64)).cuda()].double() - q[i].double()) ** 2).sum(1).cpu().numpy())
    print(f"q{i} list{l} len{len(dd)} seed512 {k512:.4f} listK {kall:.4f} r_final {r_final[i]:.4f} gtK {gtd.max():.4f} ourK {d[i, k-1]:.4f} cnt {cnt[i]}")

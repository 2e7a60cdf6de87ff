"""Timeline of one shard's search (list-sharded index on one GPU): DADE_GPU_TIMELINE=1 events.
    DADE_GPU_TIMELINE=1 python tools/shard_profile.py config2 G r"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2411_17229_b200 as gp
from paper_2411_17229_b200 import _capi, workloads as W
from paper_2411_17229_b200.dist import plan_list_shards

cfg = W.CONFIGS[sys.argv[1]]
G, r = int(sys.argv[2]), int(sys.argv[3])
dev = gp.Device(0)
art = W.build(cfg, dev, torch.device("cuda:0"), with_gt=False, log=lambda *a: None)
idx = gp.IvfIndex(dev, cfg.dim, cfg.n, cfg.nlist, art.centroids, art.offsets, art.ids, art.storage)
if G > 1:
    owner = plan_list_shards(art.offsets, G, cfg.dim)
    idx.shard((owner == r).astype(np.uint8))
    sizes = np.diff(art.offsets.astype(np.int64))
    print(f"shard {r}/{G}: lists {(owner == r).sum()} rows {sizes[owner == r].sum()}")
dco = gp.DadeStrategy(art.transform, art.cal, cfg.delta_d, dev=dev)
art.transform.upload(dev)
dev.apply(dco)
nq, k = art.q_raw.shape[0], cfg.k
keys = torch.empty((nq, k), dtype=torch.int64, device="cuda")
for it in range(3):
    st = _capi.Stats()
    _capi.check(_capi.lib.dade_gpu_ivf_search_keys(dev.h, _capi.ptr(art.q_raw), nq, k, cfg.nprobe,
                                                   _capi.DEVICE_PTRS | _capi.QUERIES_RAW, _capi.ptr(keys),
                                                   __import__("ctypes").byref(st)))
    torch.cuda.synchronize()
    print(f"dco {st.total_dco} dims {st.dims_accumulated} frac {st.dims_accumulated / max(1, st.total_dco) / cfg.dim:.4f}")
rad = np.zeros(nq, np.uint32)
_capi.check(_capi.lib.dade_gpu_debug_radius(dev.h, _capi.ptr(rad), nq))
rf = rad.view(np.float32)
print("radius: inf", int(np.isinf(rf).sum()), "median", float(np.median(rf[np.isfinite(rf)])) if np.isfinite(rf).any() else None)
buf = np.zeros(16, np.uint64)
_capi.check(_capi.lib.dade_gpu_debug_counters(dev.h, _capi.ptr(buf)))
print(f"pass1 survivors {int(buf[4]) & 0xffffffff} cands {int(buf[5]) & 0xffffffff}  "
      f"pass2 survivors {int(buf[6]) & 0xffffffff} cands {int(buf[7]) & 0xffffffff}")
print(f"pass2 survivors {int(buf[3]) & 0xffffffff} cands {int(buf[3]) >> 32}")
np.save(f"gpurun_out/radius_{sys.argv[1]}_{G}_{r}_{os.environ.get('DADE_GPU_MAX_PASS', 'all')}.npy", rf)
pr = np.zeros((nq, cfg.nprobe), np.uint64)

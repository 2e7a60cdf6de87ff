"""Per-phase clock breakdown of the DCO scan on a BASELINE workload.
    DADE_GPU_PHASES=1 python tools/phase_profile.py [config1]"""
import ctypes, os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2411_17229_b200 as gp
from paper_2411_17229_b200 import _capi, workloads as W

cfg = W.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "config1"]
dev = gp.Device(0)
art = W.build(cfg, dev, torch.device("cuda:0"), with_gt=False, log=lambda *a: None)
idx = gp.IvfIndex(dev, cfg.dim, cfg.n, cfg.nlist, art.centroids, art.offsets, art.ids, art.storage)
dco = gp.DadeStrategy(art.transform, art.cal, cfg.delta_d, dev=dev)
dev.apply(dco)
q = art.q_raw.contiguous()
nq, k = q.shape[0], cfg.k
oi = torch.empty((nq, k), dtype=torch.int32, device="cuda")
od = torch.empty((nq, k), dtype=torch.float32, device="cuda")
oc = torch.empty((nq,), dtype=torch.int32, device="cuda")
torch.cuda.synchronize()
for it in range(3):
    dev.set_profiling(True)
    st = _capi.Stats()
    _capi.check(_capi.lib.dade_gpu_ivf_search(dev.h, _capi.ptr(q), nq, k, cfg.nprobe,
                                              _capi.QUERIES_RAW | _capi.DEVICE_PTRS, _capi.ptr(oi), _capi.ptr(od),
                                              _capi.ptr(oc), ctypes.byref(st)))
    scan_ms, scan_bytes, total_ms = dev.last_scan_profile()
    filt_ms, n_filt = dev.last_filter_profile()
    buf = np.zeros(16, np.uint64)
    _capi.check(_capi.lib.dade_gpu_debug_counters(dev.h, _capi.ptr(buf)))
    ph = buf[8:13].astype(np.float64)
    if os.environ.get("DADE_GPU_DEBUG") == "1":
        print("  filter violations:", int(buf[3]))
    print(f"  pass1 survivors {int(buf[4]) & 0xffffffff} cands {int(buf[5]) & 0xffffffff}  "
          f"pass2 survivors {int(buf[6]) & 0xffffffff} cands {int(buf[7]) & 0xffffffff}")
    if os.environ.get("DADE_GPU_DEBUG") == "3":
        print(f"  merges {int(buf[3])} merged-cands {int(buf[4])} filter-kept {int(buf[5])} ckpt0-survivors {int(buf[6])}")
    names = ["wait+barrier", "dense", "epilogue", "survivors", "merges"]
    tot = ph.sum()
    print(f"scan {scan_ms:.3f} ms total {total_ms:.3f} ms dco {st.total_dco} dims {st.dims_accumulated} "
          f"frac {st.dims_accumulated / max(1, st.total_dco) / cfg.dim:.4f} "
          f"filter {filt_ms:.3f} ms / {n_filt}")
    if os.environ.get("DADE_GPU_PHASES") == "1":
        if os.environ.get("DADE_GPU_NO_UMMA") == "1":
            for p in range(3):
                a, b = int(buf[8 + 2 * p]), int(buf[9 + 2 * p])
                print(f"  filter pass {p}: tiles {a >> 32} with-kept {a & 0xffffffff} kept pairs {b}")
        else:
            c = [int(x) for x in buf[8:16]]
            ncta = 148
            us = lambda x: x / ncta / 1.9e3
            print(f"  umma pass 2 per CTA: items {c[0] / ncta:.1f} stage {us(c[1]):.1f} us | mma wait: bready "
                  f"{us(c[2]):.1f} accempty {us(c[3]):.1f} afull {us(c[4]):.1f} us | epi warp0 wait: meta "
                  f"{us(c[5]):.1f} acc {us(c[6]):.1f} us | tma wait aempty {us(c[7]):.1f} us")
    if False and tot:
        print("  " + "  ".join(f"{n} {100 * v / tot:.1f}%" for n, v in zip(names, ph)))

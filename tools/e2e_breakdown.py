"""Where the end-to-end (host buffers) time of one search goes (diagnostic).
    python tools/e2e_breakdown.py [config1]"""
import os, sys, time
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
nq, k = art.q_raw.shape[0], cfg.k
qh = torch.empty((nq, cfg.dim), dtype=torch.float32, pin_memory=True)
qh.copy_(art.q_raw.cpu())
ih = torch.empty((nq, k), dtype=torch.int32, pin_memory=True)
dh = torch.empty((nq, k), dtype=torch.float32, pin_memory=True)
ch = torch.empty((nq,), dtype=torch.int32, pin_memory=True)
qd = art.q_raw.contiguous()
idd = torch.empty((nq, k), dtype=torch.int32, device="cuda")
ddd = torch.empty((nq, k), dtype=torch.float32, device="cuda")
cdd = torch.empty((nq,), dtype=torch.int32, device="cuda")


def host():
    _capi.check(_capi.lib.dade_gpu_ivf_search(dev.h, _capi.ptr(qh), nq, k, cfg.nprobe, _capi.QUERIES_RAW,
                                              _capi.ptr(ih), _capi.ptr(dh), _capi.ptr(ch), None))


def device():
    _capi.check(_capi.lib.dade_gpu_ivf_search(dev.h, _capi.ptr(qd), nq, k, cfg.nprobe,
                                              _capi.QUERIES_RAW | _capi.DEVICE_PTRS, _capi.ptr(idd),
                                              _capi.ptr(ddd), _capi.ptr(cdd), None))
    torch.cuda.synchronize()


flush = torch.empty(512 << 18, dtype=torch.float32, device="cuda")
FLUSH = os.environ.get("FLUSH", "1") == "1"


def timeit(f, n=10):
    for _ in range(3):
        f()
    ts = []
    for _ in range(n):
        if FLUSH:
            flush.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        f()
        ts.append(time.perf_counter() - t0)
    return 1e3 * float(np.median(ts))


print(f"host-buffer search   {timeit(host):.3f} ms (wall)")
print(f"device-buffer search {timeit(device):.3f} ms (wall, incl. final sync)")
qd2 = torch.empty_like(qd)
print(f"H2D queries alone    {timeit(lambda: (qd2.copy_(qh, non_blocking=True), torch.cuda.synchronize())):.3f} ms")
print(f"D2H results alone    {timeit(lambda: (ih.copy_(idd, non_blocking=True), dh.copy_(ddd, non_blocking=True), ch.copy_(cdd, non_blocking=True), torch.cuda.synchronize())):.3f} ms")
# device-side spans of one host-buffer search (events e0 -> e3 include the H2D and D2H)
dev.set_profiling(True)
for name, f in (("host-buffer", host), ("device-buffer", device)):
    for _ in range(3):
        if FLUSH:
            flush.zero_()
        torch.cuda.synchronize()
        f()
    scan_ms, _, total_ms = dev.last_scan_profile()
    print(f"{name}: device span start->end {total_ms:.3f} ms (scan {scan_ms:.3f} ms)")
dev.set_profiling(False)

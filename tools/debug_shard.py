"""Bisect a sharded-search failure: shard r of G on one GPU, FD and ADS, per env variant.
    python tools/debug_shard.py G"""
import os, sys, subprocess
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
G = int(sys.argv[1]) if len(sys.argv) > 1 else 3
if len(sys.argv) > 2:
    import numpy as np, torch
    import paper_2411_17229_b200 as gp
    from paper_2411_17229_b200 import _capi
    from paper_2411_17229_b200.dist import plan_list_shards
    g = np.random.default_rng(31 + G)
    dim, n, nq, nlist, k, npb = 64, 30000, 700, 48, 20, 8
    centers = g.standard_normal((nlist, dim)) * 3
    assign = g.integers(0, nlist, n)
    data = (centers[assign] + g.standard_normal((n, dim)) * np.linspace(1.5, 0.2, dim)).astype(np.float32)
    order = np.lexsort((np.arange(n), assign))
    offsets = np.zeros(nlist + 1, np.uint32)
    np.add.at(offsets, assign + 1, 1)
    offsets = np.cumsum(offsets).astype(np.uint32)
    cent = np.stack([data[assign == c].mean(0) for c in range(nlist)]).astype(np.float32)
    qs = (data[g.integers(0, n, nq)] + 0.3 * g.standard_normal((nq, dim))).astype(np.float32)
    owner = plan_list_shards(offsets, G, dim)
    qd = torch.from_numpy(qs).cuda()
    kind, r = sys.argv[2], int(sys.argv[3])
    d = gp.Device(0)
    idx = gp.IvfIndex(d, dim, n, nlist, cent, offsets, order.astype(np.uint32), data[order])
    idx.shard((owner == r).astype(np.uint8))
    d.apply(gp.FdScanningStrategy(dim) if kind == "fd" else gp.AdsamplingStrategy(dim, 16, 1.5, dev=d))
    keys = torch.empty((nq, k), dtype=torch.int64, device="cuda")
    _capi.check(_capi.lib.dade_gpu_ivf_search_keys(d.h, _capi.ptr(qd), nq, k, npb, _capi.DEVICE_PTRS,
                                                   _capi.ptr(keys), None))
    torch.cuda.synchronize()
    print("ok")
    sys.exit(0)
variants = ["", "DADE_GPU_NO_SEED=1", "DADE_GPU_NO_STREAM=1", "DADE_GPU_NO_UMMA=1", "DADE_GPU_NO_QSLOTS=1",
            "DADE_GPU_SEED_NP=1", "DADE_GPU_NO_TC_COARSE=1"]
for kind in ("fd", "ads"):
    for r in range(G):
        for v in variants:
            env = dict(os.environ)
            if v:
                a, b = v.split("=")
                env[a] = b
            env["CUDA_LAUNCH_BLOCKING"] = "1"
            p = subprocess.run([sys.executable, __file__, str(G), kind, str(r)], env=env, capture_output=True, text=True)
            msg = p.stdout.strip().splitlines()[-1:] if p.returncode == 0 else p.stderr.strip().splitlines()[-1:]
            print(kind, r, v or "default", p.returncode, msg, flush=True)

"""Rotation kernel alone at the BASELINE query shapes (ncu target):
    python tools/rotate_probe.py [nq dim ...]   (default 10000 256 1000 960)"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main(shapes):
    import numpy as np
    import torch

    import paper_2411_17229_b200 as gp
    from paper_2411_17229_b200 import _capi
    dev = gp.Device(0)
    for nq, dim in shapes:
        g = np.random.default_rng(dim)
        q_, _ = np.linalg.qr(g.standard_normal((dim, dim)))
        t = gp.OrthoTransform(dim, 0, np.zeros(dim), np.ones(dim), np.ascontiguousarray(q_.T).reshape(-1))
        t.upload(dev)
        x = torch.randn(nq, dim, device="cuda") * 4
        y = torch.empty_like(x)
        dev.set_stream(torch.cuda.current_stream().cuda_stream)
        run = lambda: _capi.check(_capi.lib.dade_gpu_rotate(dev.h, _capi.ptr(x), nq, _capi.ptr(y), _capi.DEVICE_PTRS))
        for _ in range(3):
            run()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            run()
        e1.record()
        torch.cuda.synchronize()
        print(f"rotate nq={nq} dim={dim}: {e0.elapsed_time(e1) / 20 * 1e3:.1f} us", flush=True)
        dev.set_stream(None)


if __name__ == "__main__":
    a = [int(v) for v in sys.argv[1:]] or [10000, 256, 1000, 960]
    main(list(zip(a[0::2], a[1::2])))

"""H2D bandwidth of 10 MiB from differently allocated pinned host buffers (diagnostic):
torch pin_memory, cudaHostAlloc (default / write-combined), cudaHostRegister of malloc'd memory."""
import ctypes, time, glob, os
import numpy as np
import torch

lib = None
for cand in ["/usr/local/cuda/lib64/libcudart.so"] + glob.glob("/usr/local/cuda/lib64/libcudart.so.*"):
    try:
        lib = ctypes.CDLL(cand)
        break
    except OSError:
        pass
n = 10 << 20
torch.cuda.init()
dst = torch.empty(n // 4, dtype=torch.float32, device="cuda")


def bench(name, t):
    ts = []
    for i in range(40):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        dst.copy_(t, non_blocking=True)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    ts = sorted(ts[5:])
    print(f"{name:34s} med {ts[len(ts)//2]*1e3:.3f} ms -> {n/ts[len(ts)//2]/1e9:.1f} GB/s  (pinned={t.is_pinned()})")


a = torch.empty(n // 4, dtype=torch.float32, pin_memory=True)
a.fill_(1)
bench("torch pin_memory", a)
b = torch.empty(n // 4, dtype=torch.float32).pin_memory()
bench("torch .pin_memory() copy", b)
for flags, nm in ((0, "cudaHostAlloc default"), (4, "cudaHostAlloc write-combined"), (2, "cudaHostAlloc mapped")):
    p = ctypes.c_void_p()
    rc = lib.cudaHostAlloc(ctypes.byref(p), ctypes.c_size_t(n), ctypes.c_uint(flags))
    buf = (ctypes.c_char * n).from_address(p.value)
    t = torch.frombuffer(buf, dtype=torch.float32)
    t.fill_(1)
    bench(f"{nm} (rc={rc})", t)
arr = np.ones(n // 4, dtype=np.float32)
rc = lib.cudaHostRegister(ctypes.c_void_p(arr.ctypes.data), ctypes.c_size_t(n), ctypes.c_uint(0))
bench(f"cudaHostRegister(numpy) rc={rc}", torch.from_numpy(arr))
pg = 2 << 20
raw = np.ones(n // 4 + pg // 4, dtype=np.float32)
off = (-raw.ctypes.data) % pg // 4
al = raw[off:off + n // 4]
rc = lib.cudaHostRegister(ctypes.c_void_p(al.ctypes.data), ctypes.c_size_t(n), ctypes.c_uint(0))
bench(f"cudaHostRegister(2M-aligned) rc={rc}", torch.from_numpy(al))
bench("torch pin_memory again", a)

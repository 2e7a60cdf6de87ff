"""H2D/D2H bandwidth of pinned buffers under different CPU affinities (diagnostic)."""
import os, time, subprocess, sys
import torch
import pynvml
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
words = pynvml.nvmlDeviceGetCpuAffinity(h, 64)
cpus = [w * 64 + b for w, x in enumerate(words) for b in range(64) if x >> b & 1]
print("gpu0 cpu affinity:", cpus[:4], "...", cpus[-4:], len(cpus), "of", os.cpu_count())
try:
    print(subprocess.run(["nvidia-smi", "topo", "-m"], capture_output=True, text=True).stdout)
except Exception as e:
    print(e)
mode = sys.argv[1] if len(sys.argv) > 1 else "none"
allc = set(range(os.cpu_count()))
if mode == "near":
    os.sched_setaffinity(0, cpus)
elif mode == "far":
    os.sched_setaffinity(0, sorted(allc - set(cpus)) or sorted(allc))
print("mode", mode, "running on", len(os.sched_getaffinity(0)), "cpus")
n = 10 << 20
hb = torch.empty(n // 4, dtype=torch.float32, pin_memory=True)
hb.fill_(1.0)
db = torch.empty(n // 4, dtype=torch.float32, device="cuda")
for name, f in (("H2D", lambda: db.copy_(hb, non_blocking=True)), ("D2H", lambda: hb.copy_(db, non_blocking=True))):
    ts = []
    for i in range(30):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        f()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    ts.sort()
    print(f"{name} 10 MiB: min {ts[0]*1e3:.3f} ms  med {ts[len(ts)//2]*1e3:.3f} ms  -> {n/ts[len(ts)//2]/1e9:.1f} GB/s")

"""Summarise an ncu launch-list CSV (gpu__time_duration.sum): the last search's kernels.
    python tools/launches.py gpurun_out/launches.csv [anchor-kernel]"""
import csv, re, sys

rows = list(csv.reader(open(sys.argv[1])))
anchor = sys.argv[2] if len(sys.argv) > 2 else "rotate"
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
ks = [(r[ki], float(r[vi].replace(",", ""))) for r in rows[hi + 1:] if len(r) > vi]
idx = [i for i, (k, _) in enumerate(ks) if anchor in k]
last = ks[idx[-1]:]
tot = 0.0
for k, v in last:
    tot += v
    print(f"{v / 1000:8.1f} us  {re.sub(r'dade_gpu::|<unnamed>::|[(].*', '', k)[:60]}")
print(f"total {tot / 1000:.1f} us")

"""Sum an ncu launch-list CSV per kernel (diagnostic): python tools/launch_sum.py file.csv [divisor]"""
import collections, csv, re, sys
rows = list(csv.reader(open(sys.argv[1])))
div = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
agg = collections.OrderedDict()
for r in rows[hi + 1:]:
    if len(r) > vi:
        k = re.sub(r"dade_gpu::|\(anonymous namespace\)::|<unnamed>::|[(].*", "", r[ki])[:48]
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += float(r[vi].replace(",", ""))
for k, (n, v) in agg.items():
    print(f"{v / 1e3 / div:10.1f} us  x{n / div:<6.1f} {k}")

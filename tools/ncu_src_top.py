"""Top stall lines of an ncu --page source --csv export (SASS view), with the
three largest stall reasons, and per-opcode sample totals.
    python tools/ncu_src_top.py src.csv [n]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n_top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
hi = [i for i, r in enumerate(rows) if "Source" in r and "Address" in r][0]
h = rows[hi]
data = [dict(zip(h, r)) for r in rows[hi + 1:] if len(r) == len(h)]


def f(x):
    try:
        return float(x.replace(",", ""))
    except ValueError:
        return 0.0


S = "Warp Stall Sampling (All Samples)"
tot = sum(f(d[S]) for d in data)
print(f"total samples {tot:.0f}")
for i, d in sorted(enumerate(data), key=lambda x: -f(x[1][S]))[:n_top]:
    st = sorted(((k[6:], f(d[k])) for k in h if k.startswith("stall_") and "Not Issued" not in k and f(d[k]) > 0),
                key=lambda x: -x[1])[:3]
    print(f"{i:6d} {f(d[S]):6.0f} {d['Source'][:64]:64s} {st}")
agg, ex = collections.Counter(), collections.Counter()
for d in data:
    ops = [o for o in d["Source"].split() if not o.startswith("@")]
    op = ops[0] if ops else "?"
    agg[op] += f(d[S])
    ex[op] += f(d["Instructions Executed"])
for k, v in agg.most_common(15):
    print(f"{k:28s} samples {v:7.0f}  inst {ex[k]:12.0f}")

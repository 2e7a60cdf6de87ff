"""Top SASS lines by warp-stall samples of one kernel launch in an .ncu-rep (diagnostic).
    python tools/ncu_top.py report.ncu-rep [kernel-regex] [n] [launch-skip]"""
import csv, io, subprocess, sys

rep = sys.argv[1]
kern = sys.argv[2] if len(sys.argv) > 2 else ""
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
skip = sys.argv[4] if len(sys.argv) > 4 else "0"
cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "--launch-skip", skip,
       "--launch-count", "1"]
if kern:
    cmd += ["--kernel-name", "regex:" + kern]
out = subprocess.run(cmd, capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
data = [r for r in rows[2:] if len(r) == len(h)]
i_s = h.index("Warp Stall Sampling (All Samples)")
ie = h.index("Instructions Executed")
stall = [j for j, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
num = lambda x: int(x) if x.isdigit() else 0
tot = sum(num(r[i_s]) for r in data)
agg = {}
for r in data:
    for j in stall:
        agg[h[j]] = agg.get(h[j], 0) + num(r[j])
print("samples", tot, "inst", sum(num(r[ie]) for r in data))
print(sorted(agg.items(), key=lambda x: -x[1])[:8])
for r in sorted(data, key=lambda r: -num(r[i_s]))[:n]:
    st = sorted(((num(r[j]), h[j][6:]) for j in stall), reverse=True)[:2]
    print(r[0][-5:], r[i_s].rjust(5), r[ie].rjust(9), r[1][:58].ljust(58), st)

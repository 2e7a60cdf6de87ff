"""Warp-stall samples per CUDA source line of one kernel in an .ncu-rep (diagnostic).
    python tools/ncu_lines.py report.ncu-rep kernel-regex [n]"""
import csv, io, subprocess, sys

rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "--launch-count", "1",
                      "--kernel-name", "regex:" + kern], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
res, path, hdr = [], "", None
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        path = r[1].split("/")[-1]
    elif r and r[0] == "Line No":
        hdr = r
    elif hdr and r and r[0].isdigit() and len(r) >= len(hdr):
        x = len(r) - len(hdr)  # unescaped quotes in the source text split it into extra fields
        s = int(r[4 + x]) if r[4 + x].isdigit() else 0
        e = int(r[7 + x]) if r[7 + x].isdigit() else 0
        res.append((s, e, f"{path}:{r[0]}", ",".join(r[1:2 + x]).strip()[:80]))
tot = sum(x[0] for x in res) or 1
print(f"samples {tot}")
for s, e, loc, src in sorted(res, reverse=True)[:n]:
    print(f"{100 * s / tot:5.1f}%  {e:>10}  {loc:16s} {src}")

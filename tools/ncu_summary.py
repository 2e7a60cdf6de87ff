"""Per-launch summary of an ncu --set full report as JSON (profiles/ summaries).
    python tools/ncu_summary.py report.ncu-rep out.json [source-description]"""
import csv, io, json, subprocess, sys

rep, out = sys.argv[1], sys.argv[2]
src = sys.argv[3] if len(sys.argv) > 3 else ""
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, units = rows[0], rows[1]
want = {
    "us": ("gpu__time_duration.sum", 1e-3),
    "dram_read_MB": ("dram__bytes_read.sum", None),
    "dram_write_MB": ("dram__bytes_write.sum", None),
    "dram_pct_peak": ("dram__throughput.avg.pct_of_peak_sustained_elapsed", 1),
    "sm_throughput_pct": ("sm__throughput.avg.pct_of_peak_sustained_elapsed", 1),
    "fma_pipe_pct_active": ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", 1),
    "fp64_pipe_pct_active": ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", 1),
    "tensor_pipe_pct_active": ("sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active", 1),
    "issue_active_pct": ("sm__issue_active.avg.pct_of_peak_sustained_active", 1),
    "achieved_occupancy_pct": ("sm__warps_active.avg.pct_of_peak_sustained_active", 1),
    "l2_hit_pct": ("lts__t_sector_hit_rate.pct", 1),
    "inst": ("smsp__inst_executed.sum", 1),
    "registers": ("launch__registers_per_thread", 1),
}
scale = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3, "usecond": 1.0, "msecond": 1e3, "nsecond": 1e-3}
res = []
for r in rows[2:]:
    if len(r) != len(h):
        continue
    d = {"kernel": r[h.index("Kernel Name")].split("(")[0].split("::")[-1]}
    for k, (m, f) in want.items():
        if m not in h:
            continue
        i = h.index(m)
        try:
            v = float(r[i].replace(",", ""))
        except ValueError:
            continue
        u = units[i]
        if k.endswith("_MB") or k == "us":
            v *= scale.get(u, 1.0)
        d[k] = round(v, 3)
    res.append(d)
json.dump({"source": src, "launches": res}, open(out, "w"), indent=1)
for d in res:
    print(d)

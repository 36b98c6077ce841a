"""Summaries for profiles/: an ncu launch list (--metrics gpu__time_duration.sum
--csv) aggregated per kernel, and selected raw metrics of an `ncu --set full`
report, one line per profiled launch.

    python tools/summarize_ncu.py LAUNCHES.csv REPORT.ncu-rep OUT_PREFIX "command note"
"""
import collections
import csv
import io
import subprocess
import sys

launches, report, prefix, note = sys.argv[1:5]
rows = [r for r in csv.reader(open(launches)) if len(r) > 5]
h = rows[0]
ik, iv = h.index("Kernel Name"), h.index("Metric Value")
agg = collections.defaultdict(list)
for r in rows[1:]:
    agg[r[ik][:70]].append(float(r[iv].replace(",", "")) / 1e3)  # ns -> us
with open(prefix + "_launches.csv", "w") as f:
    f.write(f"# ncu launch list, gpu__time_duration.sum, --clock-control none (cold-cache, "
            f"serialised: compare SHARES); {note}\n")
    f.write("kernel,launches,total_us,mean_us\n")
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        f.write(f"\"{k}\",{len(v)},{sum(v):.1f},{sum(v) / len(v):.1f}\n")
out = subprocess.run(["ncu", "-i", report, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
r = list(csv.reader(io.StringIO(out)))
h, units = r[0], r[1]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "smsp__inst_executed.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.sum.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.sum.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size"]
ikn = h.index("Kernel Name")
lines = [f"# ncu --set full --clock-control none, one launch per kernel; {note}",
         "# columns: " + ", ".join(f"{w} [{units[h.index(w)]}]" for w in want if w in h)]
for row in r[2:]:
    lines.append(row[ikn][:60] + " | " + " | ".join(row[h.index(w)] for w in want if w in h))
open(prefix + "_ncu_summary.txt", "w").write("\n".join(lines) + "\n")
print("\n".join(lines))

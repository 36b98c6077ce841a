"""Turn gpurun_out/{launches.csv,synth_full.ncu-rep} (tools/profile_synth_round.sh)
into profiles/r1_synth_launches_summary.csv and r1_synth_ncu_full_summary.txt."""
import collections
import csv
import io
import os
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1] if len(sys.argv) > 1 else "current kernels"
KS = ("balance_kernel", "decompose_kernel", "sort_kernel")
rows = [r for r in csv.reader(open(os.path.join(REPO, "gpurun_out/launches.csv"))) if len(r) > 5]
h = rows[0]
ik, iv = h.index("Kernel Name"), h.index("Metric Value")
agg = collections.defaultdict(list)
for r in rows[1:]:
    name = r[ik].split("(")[0].split("::")[-1].split("<")[0]
    if name in KS:
        agg[name].append(float(r[iv].replace(",", "")) / 1e6)
tot = sum(sum(v) for v in agg.values())
with open(os.path.join(REPO, "profiles/r1_synth_launches_summary.csv"), "w") as f:
    f.write("# ncu launch list (gpu__time_duration.sum, --clock-control none; cold-cache, serialised: compare SHARES)\n")
    f.write(f"# command: python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e   (config 5: n=128 x m=8, batch 1000; {tag})\n")
    f.write("kernel,launches,total_ms,mean_ms,share_of_synthesis\n")
    for k in KS:
        v = agg[k]
        f.write(f"{k},{len(v)},{sum(v):.3f},{sum(v)/len(v):.4f},{sum(v)/tot:.4f}\n")
out = subprocess.run(["ncu", "-i", os.path.join(REPO, "gpurun_out/synth_full.ncu-rep"), "--page", "raw",
                      "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(out)))
h, units = r[0], r[1]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__grid_size", "launch__block_size",
        "smsp__inst_executed.sum", "sm__inst_executed.avg.per_cycle_active"]
ikn = h.index("Kernel Name")
lines = ["# ncu --set full --clock-control none, one launch per kernel",
         f"# command: python tools/profile_synth.py --n 128 --batch 1000 --reps 1  (config 5: n=128 x m=8, batch 1000; {tag})"]
for row in r[2:]:
    name = row[ikn].split("(")[0].split("::")[-1].split("<")[0]
    lines.append(name + ": " + ", ".join(f"{w}={row[h.index(w)]} {units[h.index(w)]}" for w in want if w in h))
lines.append("balance_kernel algorithmic bytes 16*G^2*B = 16.78 GB")
lines.append("decompose_kernel algorithmic bytes 16*n^2 + n_raw*(8+9n) per matrix = 18.9 GB per batch "
             "(stage outputs dominate); a latency chain, see r1_decompose_ncu_lines.txt")
open(os.path.join(REPO, "profiles/r1_synth_ncu_full_summary.txt"), "w").write("\n".join(lines) + "\n")
print("\n".join(lines))

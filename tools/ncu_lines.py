"""Aggregate ncu warp-stall samples of one kernel per CUDA source line.

    python tools/ncu_lines.py REPORT.ncu-rep LIB.so KERNEL_SUBSTRING [top]

ncu's own CUDA-source page carries no metrics for this build (the box path
differs), so this maps the SASS page's per-instruction samples to source
lines with the -lineinfo tables (`nvdisasm -g -c` on the cubin of LIB.so).
"""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile


def sass_samples(report: str, kernel: str = ""):
    """[(offset, sass text, stall samples, instructions executed)] of the
    first kernel matching `kernel` in the report."""
    cmd = ["ncu", "-i", report, "--page", "source", "--csv", "--print-source", "sass"]
    if kernel:
        cmd += ["-k", f"regex:{kernel}"]
    out = subprocess.run(cmd, capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    hdr = rows[h]
    ia, isrc = hdr.index("Address"), hdr.index("Source")
    isamp = hdr.index("Warp Stall Sampling (All Samples)")
    iexe = hdr.index("Instructions Executed")
    data = []
    for r in rows[h + 1:]:
        if not r or not r[0].startswith("0x"):
            break
        data.append((int(r[ia], 16), r[isrc].strip(), int(r[isamp] or 0), int(r[iexe] or 0)))
    base = data[0][0]
    return [(a - base, s_, n, e) for a, s_, n, e in data]


def line_table(lib: str, kernel: str):
    tmp = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=tmp, capture_output=True)
    table = {}
    for f in os.listdir(tmp):
        if not f.endswith(".cubin"):
            continue
        txt = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(tmp, f)], capture_output=True,
                             text=True).stdout
        cur_fn, cur_line = None, None
        for line in txt.splitlines():
            if line.startswith(".text.") and line.rstrip().endswith(":"):
                cur_fn = line[6:-1]
            m = re.search(r'//## File "([^"]+)", line (\d+)', line)
            if m:
                cur_line = f"{os.path.basename(m.group(1))}:{m.group(2)}"
                continue
            m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", line)
            if m and cur_fn and kernel in cur_fn:
                table.setdefault(cur_fn, {})[int(m.group(1), 16)] = cur_line
    return table


def main():
    report, lib, kernel = sys.argv[1:4]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
    samples = sass_samples(report, kernel)
    tables = line_table(lib, kernel)
    # pick the function whose instruction count matches the ncu listing
    fn = min(tables, key=lambda k: abs(len(tables[k]) - len(samples)))
    tab = tables[fn]
    agg, ins = collections.Counter(), collections.Counter()
    for off, _, n, e in samples:
        agg[tab.get(off, "?")] += n
        ins[tab.get(off, "?")] += e
    tot = sum(agg.values()) or 1
    itot = sum(ins.values()) or 1
    print(f"{fn}: {tot} stall samples, {itot} warp instructions executed")
    print(" samples%  instr%   line")
    for k, v in agg.most_common(top):
        print(f"{100 * v / tot:7.2f}% {100 * ins[k] / itot:7.2f}%  {k}")


if __name__ == "__main__":
    main()

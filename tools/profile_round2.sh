#!/bin/bash
# Round-2 ncu evidence for the config-5 synthesis path (run on a GPU box,
# after bench.py itself has exited 0 without ncu).  Outputs in gpurun_out/.
set -x
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches.csv \
    python bench.py --steps 2 --warmup 3 --inflight 1 --no-cpu-baseline --no-e2e --no-latency \
    > gpurun_out/r2_launches.log 2>&1
ncu --set full --import-source on --clock-control none \
    -k regex:"balance_kernel|decompose_kernel|sort_kernel|strip_table|compact_" -c 7 \
    -o gpurun_out/r2_synth_full python tools/profile_synth.py --n 128 --batch 1000 --reps 1 --compact \
    > gpurun_out/r2_synth_full.log 2>&1
ncu -i gpurun_out/r2_synth_full.ncu-rep --page raw --csv > gpurun_out/r2_synth_full_raw.csv 2>&1
python tools/ncu_lines.py gpurun_out/r2_synth_full.ncu-rep paper_2505_09764_b200/libfastb200.so \
    decompose_kernel 40 > gpurun_out/r2_decompose_lines.txt 2>&1

#!/bin/bash
# Bench line + ncu evidence for the config-5 synthesis path (run on a GPU box).
# Outputs under gpurun_out/: bench_synth.json, launches.csv, synth_full.ncu-rep
set -x
python bench.py > gpurun_out/bench_synth.json 2> gpurun_out/bench_synth.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/launches.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"balance_kernel|decompose_kernel|sort_kernel" -c 3 \
    -o gpurun_out/synth_full python tools/profile_synth.py --n 128 --batch 1000 --reps 1 > gpurun_out/synth_full.log 2>&1

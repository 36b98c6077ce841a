#!/bin/bash
# What the driver runs at round end on a fresh 1-GPU box: GPU tests, smoke,
# the bench line and the reference arm (outputs in gpurun_out/re_*).
python -m pytest tests -x -q -m gpu > gpurun_out/re_pytest.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/re_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/re_smoke.log 2>&1; echo "smoke rc=$?"
python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/re_bench.json 2> gpurun_out/re_bench.err; echo "bench rc=$?"

python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/re_ref.json 2> gpurun_out/re_ref.err; echo "ref rc=$?"

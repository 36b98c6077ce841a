#!/bin/bash
# End-of-session validation + bench lines (run with gpurun --gpus 4).
set -x
python -m pytest tests -m gpu -q 2>&1 | tail -3
python -c "import __graft_entry__ as g; g.smoke()" && echo SMOKE_OK
python bench.py > gpurun_out/final_bench_n1.json 2>gpurun_out/final_bench_n1.err
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29801 bench.py --gpus 2 --steps 20 --warmup 5 2>/dev/null | grep '^{' > gpurun_out/final_bench_n2.json
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29802 bench.py --gpus 4 --steps 20 --warmup 5 2>/dev/null | grep '^{' > gpurun_out/final_bench_n4.json
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29803 bench.py --gpus 4 --steps 20 --warmup 5 --topo 4x1 2>/dev/null | grep '^{' > gpurun_out/final_bench_n4_4x1.json
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29804 bench.py --gpus 4 --steps 10 --warmup 3 --workload moe 2>/dev/null | grep '^{' > gpurun_out/final_moe_n4.json
for f in gpurun_out/final_*.json; do echo "$f"; head -c 400 "$f"; echo; done

#!/bin/bash
# fused pack -> send: A/B on one GPU, ncu launch list of it, config-3 lines at 2/4 GPUs
timeout 300 python tools/fused_pack_ab.py > gpurun_out/fp_ab.json 2> gpurun_out/fp_ab.err; tail -c 600 gpurun_out/fp_ab.json
timeout 300 python tools/fused_pack_ab.py --steps 2 > /dev/null 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/fp_ab_ncu.csv python tools/fused_pack_ab.py --steps 2 > gpurun_out/fp_ab_ncu.log 2>&1
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29811 bench.py --gpus 2 --steps 10 --warmup 3 --workload moe 2>gpurun_out/fp_moe_n2.err | grep '^{' > gpurun_out/fp_moe_n2.json
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29812 bench.py --gpus 4 --steps 10 --warmup 3 --workload moe 2>gpurun_out/fp_moe_n4.err | grep '^{' > gpurun_out/fp_moe_n4.json
for f in gpurun_out/fp_moe_n*.json; do echo $f; head -c 300 $f; echo; done

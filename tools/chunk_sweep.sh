#!/bin/bash
# config 2 at N GPUs: exec chunk-size sweep (bench --chunk), default topology
N=${1:-4}
for C in 262144 524288 1048576 2097152 1048576; do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
    --master-port 29661 bench.py --gpus $N --steps 20 --warmup 5 --chunk $C 2>/dev/null | grep '^{' | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('chunk $C', d['value'], d['exec_kernel_ms'], d['synth_and_plan_ms'], d['roofline'].get('exec_vs_fast_achievable'))"
done

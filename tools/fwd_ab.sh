#!/bin/bash
# exec forwarder-pool scale A/B (config 2, N GPUs): FASTB200_LIB per variant
N=${1:-4}; shift
for L in paper_2505_09764_b200/libfastb200.so "$@" paper_2505_09764_b200/libfastb200.so; do
  FASTB200_LIB=$L timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N \
    --master-addr 127.0.0.1 --master-port 29651 bench.py --gpus $N --steps 20 --warmup 5 2>/dev/null \
    | grep '^{' | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$L', d['value'], d['exec_kernel_ms'], d['roofline'].get('exec_vs_fast_achievable'))"
done

#!/bin/bash
# config-2 exec bandwidth vs CTAs per rank (SMs the executor occupies)
N=${1:-4}
for B in 16 32 64 96 128; do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
    --master-port 29651 bench.py --gpus $N --steps 10 --warmup 3 --blocks $B 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('blocks $B', d['value'], 'GB/s step', d['exec_kernel_ms'], 'ms exec')"
done

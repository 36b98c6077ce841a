#!/bin/bash
# config-2 exec: blocks x chunk sweep at N GPUs (topology default 2 x N/2)
N=${1:-4}; TOPO=${2:-}
for B in 128 148; do for C in 524288 1048576 2097152; do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
    --master-port 29631 bench.py --gpus $N --steps 10 --warmup 3 --blocks $B --chunk $C ${TOPO:+--topo $TOPO} 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('blocks $B chunk $C', d['value'], d['exec_kernel_ms'], d['roofline'].get('exec_vs_fast_achievable'))"
done; done

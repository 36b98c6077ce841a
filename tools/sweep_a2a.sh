#!/bin/bash
# usage: tools/sweep_a2a.sh N "blocks chunk topo" ...   (run on a GPU box)
N=$1; shift
port=29600
for cfg in "$@"; do
  set -- $cfg
  port=$((port+1))
  timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr 127.0.0.1 --master-port $port \
     bench.py --gpus $N --steps 20 --warmup 5 --blocks $1 --chunk $2 --topo $3 2>/dev/null | tail -1 | \
     python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('N=$N blocks=$1 chunk=$2 topo=$3', 'GBs', d['value'], 'exec_ms', d['exec_kernel_ms'], 'step_ms', d['ms_per_step'], 'frac', r['frac'], 'ceil', r['fast_one_tier_ceiling'], 'nccl', d['nccl_all_to_all_single']['value'])"
done

#!/bin/bash
# usage: tools/sweep_lib.sh N LIB "blocks chunk topo" ...
N=$1; LIB=$2; shift 2
port=29700
for cfg in "$@"; do
  set -- $cfg
  port=$((port+1))
  FASTB200_LIB=$LIB timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr 127.0.0.1 --master-port $port \
     bench.py --gpus $N --steps 20 --warmup 5 --blocks $1 --chunk $2 --topo $3 2>/dev/null | tail -1 | \
     python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$LIB N=$N blocks=$1 chunk=$2 topo=$3', 'GBs', d['value'], 'exec_ms', d['exec_kernel_ms'], 'frac', r['frac'], 'nccl', d['nccl_all_to_all_single']['value'], 'clk', d['clocks'].get('sm_mhz'), d['clocks'].get('reasons'))"
done

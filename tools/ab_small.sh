#!/bin/bash
# Small-message per-call latency A/B of experiment builds (run on a GPU box).
# usage: tools/ab_small.sh N lib1.so lib2.so ...
N=$1; shift
port=29700
for l in "$@"; do
  port=$((port+1))
  if [ "$l" = default ]; then unset FASTB200_LIB; else export FASTB200_LIB=$l; fi
  echo "== $l"
  timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr 127.0.0.1 \
    --master-port $port tools/small_a2a.py 2>&1 | grep -E "per call|stages us"
done

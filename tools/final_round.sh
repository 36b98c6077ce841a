#!/bin/bash
# End-of-session multi-GPU validation + bench lines (run with gpurun --gpus 4).
# Outputs: gpurun_out/fin_*.json / .log
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
python -m pytest tests/test_exec_multi.py tests/test_exec_fuzz.py -m gpu -q > gpurun_out/fin_multi_tests.log 2>&1
echo "multi-GPU tests rc=$?"; tail -2 gpurun_out/fin_multi_tests.log
run() {  # name, nproc, port, args...
  local name=$1 np=$2 port=$3; shift 3
  timeout 600 $TR --nproc-per-node $np --master-port $port bench.py --gpus $np "$@" \
      > gpurun_out/fin_$name.out 2> gpurun_out/fin_$name.err
  grep '^{' gpurun_out/fin_$name.out | tail -1 > gpurun_out/fin_$name.json
  echo "$name rc=$? $(head -c 300 gpurun_out/fin_$name.json)"
}
run a2a_n2 2 29811 --steps 20 --warmup 5
run ref_n2 2 29812 --steps 3 --warmup 1 --impl reference
run moe_n2 2 29813 --steps 20 --warmup 5 --workload moe
run a2a_n4 4 29814 --steps 20 --warmup 5
run a2a_n4_4x1 4 29815 --steps 20 --warmup 5 --topo 4x1
run moe_n4 4 29816 --steps 20 --warmup 5 --workload moe
run moe_n4_4x1 4 29817 --steps 20 --warmup 5 --workload moe --topo 4x1
run ref_n4 4 29818 --steps 3 --warmup 1 --impl reference

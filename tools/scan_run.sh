#!/bin/bash
python -m pytest tests -m gpu -q 2>&1 | tail -3
python -c "import __graft_entry__ as g; g.smoke()" && echo SMOKE_OK
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29821 bench.py --gpus 2 --steps 10 --warmup 3 --workload moe 2>gpurun_out/sc_moe_n2.err | grep '^{' > gpurun_out/sc_moe_n2.json
head -c 300 gpurun_out/sc_moe_n2.json; echo
timeout 300 python tools/fused_pack_ab.py --steps 2 > /dev/null 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:moe_route --log-file gpurun_out/sc_ncu.csv python tools/fused_pack_ab.py --steps 2 > gpurun_out/sc_ncu.log 2>&1

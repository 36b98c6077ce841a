set -x
python -m pytest tests -q -m gpu -x 2>&1 | tail -4
for T in 2x2 4x1; do timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29521 bench.py --gpus 4 --steps 20 --warmup 5 --workload alltoallv --topo $T --no-cpu-baseline 2>&1 | grep '^{' > gpurun_out/a2a_4_$T.json; tail -c 600 gpurun_out/a2a_4_$T.json; echo; done
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29522 bench.py --gpus 2 --steps 20 --warmup 5 --workload alltoallv --topo 2x1 --no-cpu-baseline 2>&1 | grep '^{' > gpurun_out/a2a_2_2x1.json; tail -c 600 gpurun_out/a2a_2_2x1.json

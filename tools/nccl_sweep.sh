#!/bin/bash
# NCCL all_to_all_single on the config-2 traffic under several NCCL knob
# settings (a fair bar for the FAST executor).  usage: tools/nccl_sweep.sh N
N=${1:-4}
run() {
  env "$@" timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N \
    --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus $N --steps 20 --warmup 5 \
    --nccl-only 2>/dev/null | tail -1
}
run X=1
run NCCL_NCHANNELS_PER_PEER=32
run NCCL_NCHANNELS_PER_PEER=32 NCCL_MIN_P2P_NCHANNELS=32 NCCL_MAX_P2P_NCHANNELS=32
run NCCL_NCHANNELS_PER_PEER=32 NCCL_MIN_P2P_NCHANNELS=64 NCCL_MAX_P2P_NCHANNELS=64
run NCCL_NCHANNELS_PER_PEER=64 NCCL_MIN_P2P_NCHANNELS=64 NCCL_MAX_P2P_NCHANNELS=64
run NCCL_NCHANNELS_PER_PEER=32 NCCL_MIN_P2P_NCHANNELS=64 NCCL_MAX_P2P_NCHANNELS=64 NCCL_P2P_NVL_CHUNKSIZE=1048576
run NCCL_NCHANNELS_PER_PEER=16 NCCL_MIN_P2P_NCHANNELS=64 NCCL_MAX_P2P_NCHANNELS=64

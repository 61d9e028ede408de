#!/bin/bash
# N-GPU check: multi-GPU tests + benches (run under gpurun --gpus N)
N=${1:-2}
OUT=${2:-gpurun_out/nrun}
mkdir -p $(dirname $OUT)
timeout 600 python -m pytest tests/test_gpu_multi.py -q -p no:cacheprovider > ${OUT}_multi.txt 2>&1
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511"
timeout 300 $TR bench.py --gpus $N --steps 30 --warmup 5 --trace > ${OUT}_bench.txt 2>&1
timeout 300 $TR bench.py --gpus $N --steps 30 --warmup 5 --workload alexnet-dense --no-csc --trace >> ${OUT}_bench.txt 2>&1

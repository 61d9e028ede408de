#!/bin/bash
# CSC exchange-overlap knobs at N GPUs: CTA size x grid cap
N=${1:-2}; OUT=${2:-gpurun_out/cscab}
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2953$N"
for wl in alexnet-csc resnet50-csc; do
  for cfg in "0 64" "256 64" "256 128" "256 32"; do
    set -- $cfg
    GF_CSC_XTHREADS=$1 GF_CSC_XBLOCKS=$2 timeout 300 $TR bench.py --gpus $N --steps 30 --warmup 5 --workload $wl --no-e2e --no-cpu-baseline > ${OUT}_n${N}_${wl}_t$1_b$2.txt 2>&1
  done
done

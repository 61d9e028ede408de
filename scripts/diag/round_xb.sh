#!/bin/bash
# N=4 routed CSC exchange: its CTA budget beside the packing (GF_CSC_XBLOCKS x GF_CSC_XTHREADS)
P=gpurun_out/r2xb
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29647"
B="--gpus 4 --steps 30 --warmup 5 --no-csc --no-e2e --no-cpu-baseline"
for wl in resnet50-csc alexnet-csc; do
  for cfg in "64 256" "128 256" "148 512" "32 512"; do
    set -- $cfg
    GF_CSC_XBLOCKS=$1 GF_CSC_XTHREADS=$2 timeout 150 $TR bench.py $B --workload $wl > ${P}_${wl}_b$1_t$2.txt 2>&1
  done
done

#!/bin/bash
# A/B of the rspush variants: unpack fused into rsp_kernel (GF_FUSE_UNPACK) x routed pack split
# into local / remote grids (GF_PUSH_SPLIT), at N GPUs. usage: rspush_ab.sh N OUTPREFIX [workloads]
N=${1:-2}; OUT=${2:-gpurun_out/ab}; WLS=${3:-"resnet50-dense alexnet-dense"}
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2952$N"
for wl in $WLS; do
  for fu in 1 0; do
    for sp in 0 1; do
      GF_FUSE_UNPACK=$fu GF_PUSH_SPLIT=$sp timeout 300 $TR bench.py --gpus $N --steps 30 --warmup 5 --workload $wl --no-csc --no-e2e --no-cpu-baseline --trace > ${OUT}_n${N}_${wl}_fu${fu}_sp${sp}.txt 2>&1
    done
  done
done

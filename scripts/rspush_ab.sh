#!/bin/bash
# A/B of the rspush variants at N GPUs: routed pack form (TMA-staged / register stores) x
# unpack (fused into rsp_kernel / separate launch).  usage: rspush_ab.sh N OUTPREFIX [workloads]
N=${1:-2}; OUT=${2:-gpurun_out/ab}; WLS=${3:-"resnet50-dense alexnet-dense"}
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29512"
for wl in $WLS; do
  for tma in 1 0; do
    for fu in 1 0; do
      GF_PACK_TMA=$tma GF_FUSE_UNPACK=$fu timeout 300 $TR bench.py --gpus $N --steps 30 --warmup 5 --workload $wl --no-csc --no-e2e --trace > ${OUT}_${wl}_tma${tma}_fu${fu}.txt 2>&1
    done
  done
done

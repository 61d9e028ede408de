#!/bin/bash
# Pipelined rspush sweep: GF_PUSH_PIECES x GF_PUSH_RSP_BLOCKS at N GPUs (bench lines + trace).
# usage: pieces_sweep.sh N OUTPREFIX "P list" "B list" [workloads]
N=${1:-2}; OUT=${2:-gpurun_out/pc}; PS=${3:-"1 2 4 8"}; BS=${4:-"32 64 148"}; WLS=${5:-"resnet50-dense alexnet-dense"}
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2953$N"
for wl in $WLS; do
  for P in $PS; do
    for B in $BS; do
      [ "$P" = 1 ] && [ "$B" != "$(echo $BS | cut -d' ' -f1)" ] && continue
      GF_PUSH_PIECES=$P GF_PUSH_RSP_BLOCKS=$B timeout 300 $TR bench.py --gpus $N --steps 30 --warmup 5 --workload $wl \
        --no-csc --no-e2e --no-cpu-baseline --trace > ${OUT}_n${N}_${wl}_p${P}_b${B}.txt 2>&1
    done
  done
done

#!/bin/bash
# rsp_kernel: the fused own-segment unpack after the push sweep (GF_RSP_LATE_UNPACK) at N=2/4
P=gpurun_out/r2l
GF_RSP_LATE_UNPACK=1 GF_FUSE_UNPACK=1 timeout 400 python -m pytest tests/test_gpu_colocated.py -q -x -p no:cacheprovider -k "rspush or resnet50_full or alexnet_4rank" > ${P}_colo.txt 2>&1
B="--steps 30 --warmup 5 --no-csc --no-e2e --no-cpu-baseline --trace --dense-mode rspush"
for N in 2 4; do
  TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2961$N"
  for wl in resnet50-dense alexnet-dense; do
    for cfg in "1 0" "1 1" "0 0"; do
      set -- $cfg
      GF_FUSE_UNPACK=$1 GF_RSP_LATE_UNPACK=$2 timeout 200 $TR bench.py --gpus $N $B --workload $wl > ${P}_n${N}_${wl}_fu$1_late$2.txt 2>&1
    done
  done
done

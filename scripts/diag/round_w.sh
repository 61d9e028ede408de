#!/bin/bash
# 2-GPU box: the one-kernel pipelined dense step (parity colocated + N=2 sweep), CSC launch order A/B, NVLink ncu
P=gpurun_out/r2w
timeout 600 python -m pytest tests/test_gpu_colocated.py -q -x -p no:cacheprovider -k "pipe" > ${P}_colo_pipe.txt 2>&1
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29573"
B="--gpus 2 --steps 30 --warmup 5 --no-csc --no-e2e --no-cpu-baseline --trace"
for wl in resnet50-dense alexnet-dense; do
  timeout 300 $TR bench.py $B --workload $wl --dense-mode rspush > ${P}_n2_${wl}_rspush.txt 2>&1
  for ue in 8192 16384 32768; do
    for cons in 1 2 3; do
      GF_PIPE_UE=$ue GF_PIPE_CONS=$cons timeout 300 $TR bench.py $B --workload $wl --dense-mode pipe > ${P}_n2_${wl}_pipe_u${ue}_c${cons}.txt 2>&1
    done
  done
done
for wl in resnet50-csc alexnet-csc; do
  for o in 0 1; do
    GF_CSC_ORDER=$o timeout 300 $TR bench.py $B --workload $wl > ${P}_n2_${wl}_order${o}.txt 2>&1
  done
done
bash scripts/diag/ncu_nvl.sh ${P}_nvl 2 "resnet50-dense" "rspush pipe push csc-push" > ${P}_nvl.txt 2>&1

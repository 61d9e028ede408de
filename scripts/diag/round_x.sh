#!/bin/bash
# 2-GPU box: pipe kernel with backoff polling (parity + sweep), NVLink ncu of every N>1 kernel
P=gpurun_out/r2x
timeout 600 python -m pytest tests/test_gpu_colocated.py -q -x -p no:cacheprovider -k "pipe" > ${P}_colo_pipe.txt 2>&1
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29574"
B="--gpus 2 --steps 30 --warmup 5 --no-csc --no-e2e --no-cpu-baseline --trace"
for wl in resnet50-dense alexnet-dense; do
  for ue in 8192 32768; do
    for cons in 1 2 3; do
      GF_PIPE_UE=$ue GF_PIPE_CONS=$cons timeout 200 $TR bench.py $B --workload $wl --dense-mode pipe > ${P}_n2_${wl}_pipe_u${ue}_c${cons}.txt 2>&1
    done
  done
done
bash scripts/diag/ncu_nvl.sh ${P}_nvl 2 "resnet50-dense" "rspush pipe push pull csc-push csc-pull" > ${P}_nvl.txt 2>&1

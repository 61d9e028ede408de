#!/bin/bash
# 2-GPU box: pipelined rspush (correctness at P=4 colocated + sweep), select phases, NVLink ncu
P=gpurun_out/r2t
GF_PUSH_PIECES=4 timeout 500 python -m pytest tests/test_gpu_colocated.py -q -x -p no:cacheprovider \
  -k "rspush or resnet50_full or alexnet_4rank" > ${P}_colo_p4.txt 2>&1
timeout 300 python -m pytest tests/test_gpu_kernels.py -q -x -p no:cacheprovider -k "select or csc" > ${P}_select.txt 2>&1
timeout 300 python bench.py --workload alexnet-csc --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --no-csc --trace > ${P}_n1_acsc.txt 2>&1
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29571"
for wl in resnet50-csc alexnet-csc; do
  timeout 300 $TR bench.py --gpus 2 --steps 30 --warmup 5 --workload $wl --no-csc --no-e2e --no-cpu-baseline --trace > ${P}_n2_${wl}.txt 2>&1
done
bash scripts/pieces_sweep.sh 2 ${P} "1 2 4 8" "32 64 148"
bash scripts/diag/ncu_nvl.sh ${P}_nvl 2 "resnet50-dense" "rspush pull push csc-push csc-pull" > ${P}_nvl.txt 2>&1

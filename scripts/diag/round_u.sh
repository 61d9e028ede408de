#!/bin/bash
# 2-GPU box: CSC (plan-driven part-1 pack, momentum update fused into the exchange) parity + benches
P=gpurun_out/r2u
timeout 600 python -m pytest tests/test_gpu_colocated.py -q -x -p no:cacheprovider -k "csc" > ${P}_colo_csc.txt 2>&1
timeout 300 python -m pytest tests/test_gpu_kernels.py -q -x -p no:cacheprovider -k "select or csc or sgd" > ${P}_kernels.txt 2>&1
timeout 300 python bench.py --workload alexnet-csc --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --no-csc --trace > ${P}_n1_acsc.txt 2>&1
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29572"
for wl in resnet50-csc alexnet-csc; do
  for cm in push pull; do
    timeout 300 $TR bench.py --gpus 2 --steps 30 --warmup 5 --workload $wl --csc-mode $cm --no-csc --no-e2e --no-cpu-baseline --trace > ${P}_n2_${wl}_${cm}.txt 2>&1
  done
done
bash scripts/diag/nvl_dbg.sh > ${P}_nvl_dbg.txt 2>&1

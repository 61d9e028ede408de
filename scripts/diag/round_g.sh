#!/bin/bash
# 4-GPU box: routed CSC exchange (pull form) parity + N=1/2/4 CSC benches, select 3-pass, world-1 CSC split
P=gpurun_out/r2g
timeout 900 python -m pytest tests/test_gpu_colocated.py tests/test_gpu_kernels.py -q -x -p no:cacheprovider -k "csc or select or sgd" > ${P}_pytest.txt 2>&1
timeout 300 python bench.py --workload alexnet-csc --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --no-csc --trace > ${P}_n1_acsc.txt 2>&1
timeout 300 python bench.py --workload resnet50-csc --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --no-csc --trace > ${P}_n1_rcsc.txt 2>&1
for N in 2 4; do
  TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2959$N"
  for wl in resnet50-csc alexnet-csc; do
    for cm in pull push; do
      timeout 300 $TR bench.py --gpus $N --steps 30 --warmup 5 --workload $wl --csc-mode $cm --no-csc --no-e2e --no-cpu-baseline --trace > ${P}_n${N}_${wl}_${cm}.txt 2>&1
    done
  done
done
timeout 600 python -m pytest tests/test_gpu_multi.py -q -x -p no:cacheprovider -k "csc" > ${P}_pytest_multi.txt 2>&1

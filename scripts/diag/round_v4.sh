#!/bin/bash
# 4-GPU final verification: cross-GPU tests + the N=2/N=4 stress, N=2/N=4 benches, NVLink ncu of the routed CSC exchange
P=gpurun_out/r2v4
timeout 1200 python -m pytest tests/test_gpu_multi.py tests/test_gpu_stress.py -m gpu -q -p no:cacheprovider -k "not colocated" > ${P}_pytest_multi.txt 2>&1; echo "rc=$?" >> ${P}_pytest_multi.txt
for N in 2 4; do
  TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2960$N"
  timeout 600 $TR bench.py --gpus $N --trace > ${P}_bench_n${N}.txt 2>&1
  for w in alexnet-dense resnet50-csc alexnet-csc; do
    timeout 400 $TR bench.py --gpus $N --steps 30 --warmup 5 --workload $w --no-csc --no-e2e --no-cpu-baseline --trace > ${P}_bench_n${N}_$w.txt 2>&1
  done
done
bash scripts/diag/ncu_nvl.sh ${P}_nvl4 4 "resnet50-dense" "csc-pull" > ${P}_nvl4.txt 2>&1
du -sh gpurun_out

#!/bin/bash
# final 4-GPU verification: colocated CSC + cross-GPU suite + N=4 stress, N=2/N=4 default bench lines
P=gpurun_out/r2z4
timeout 600 python -m pytest tests/test_gpu_colocated.py -q -p no:cacheprovider -k "csc" > ${P}_colo_csc.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_multi.py tests/test_gpu_stress.py -m gpu -q -p no:cacheprovider -k "not colocated" > ${P}_pytest_multi.txt 2>&1; echo "rc=$?" >> ${P}_pytest_multi.txt
for N in 2 4; do
  TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2963$N"
  timeout 600 $TR bench.py --gpus $N --trace > ${P}_bench_n${N}.txt 2>&1
  timeout 400 $TR bench.py --gpus $N --steps 30 --warmup 5 --workload resnet50-csc --no-csc --no-e2e --no-cpu-baseline --trace > ${P}_bench_n${N}_resnet50-csc.txt 2>&1
done

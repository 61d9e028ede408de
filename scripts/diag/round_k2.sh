#!/bin/bash
# 1-GPU: K2 without the per-vector division (U=1 / U=2 in flight): parity + N=1 CSC benches
P=gpurun_out/r2k
for u in 1 2; do
  GF_K2_U=$u timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_colocated.py -q -x -p no:cacheprovider -k "csc" > ${P}_pytest_u$u.txt 2>&1
  for w in alexnet-csc resnet50-csc; do
    GF_K2_U=$u timeout 300 python bench.py --workload $w --steps 30 --warmup 5 --no-e2e --no-cpu-baseline --no-csc > ${P}_n1_${w}_u$u.txt 2>&1
  done
done

#!/bin/bash
# 1-GPU: momentum update over the staged index space (GF_SGD_FLAT) — parity + N=1 CSC benches A/B
P=gpurun_out/r2sgd
GF_SGD_FLAT=1 timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_colocated.py -q -x -p no:cacheprovider -k "sgd or csc" > ${P}_pytest.txt 2>&1
for f in 1 0 1 0; do
  for w in alexnet-csc resnet50-csc; do
    GF_SGD_FLAT=$f timeout 300 python bench.py --workload $w --steps 30 --warmup 5 --no-e2e --no-cpu-baseline --no-csc >> ${P}_n1_${w}_flat$f.txt 2>&1
  done
done

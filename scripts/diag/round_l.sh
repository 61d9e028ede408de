#!/bin/bash
P=gpurun_out/r2l
timeout 900 python -m pytest tests/test_gflowpy.py tests/test_reference_suites.py tests/test_gpu_colocated.py -q -x -p no:cacheprovider > ${P}_tests.txt 2>&1
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29515"
for xb in 32 64; do
  for wl in alexnet-csc resnet50-csc; do
    GF_CSC_XBLOCKS=$xb timeout 300 $TR bench.py --gpus 2 --steps 30 --warmup 5 --workload $wl --no-e2e > ${P}_csc_${wl}_xb${xb}.txt 2>&1
  done
done
timeout 300 python bench.py --steps 20 --warmup 5 > ${P}_bench1.txt 2>&1
CUDA_VISIBLE_DEVICES=0 timeout 300 /usr/local/cuda/bin/ncu --set full --import-source on --clock-control none -k "regex:pack" -c 4 -f -o ${P}_pack python scripts/diag/pack_ncu.py > ${P}_pack_ncu.log 2>&1

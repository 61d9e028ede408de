#!/bin/bash
# pack_push / CSC timing probes at N=2 (diagnostic; GF_PUSH_DIAG=1 results are invalid by design)
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29514"
P=${1:-gpurun_out/probe}
for d in 0 1; do
  GF_PUSH_DIAG=$d timeout 300 $TR bench.py --gpus 2 --steps 30 --warmup 5 --no-csc --no-e2e > ${P}_diag${d}.txt 2>&1
done
for xb in 32 64 148; do
  for wl in alexnet-csc resnet50-csc; do
    GF_CSC_XBLOCKS=$xb timeout 300 $TR bench.py --gpus 2 --steps 30 --warmup 5 --workload $wl --no-e2e > ${P}_csc_${wl}_xb${xb}.txt 2>&1
  done
done

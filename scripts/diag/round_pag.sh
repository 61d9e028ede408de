#!/bin/bash
# routed CSC exchange: pulled vs pushed all-gather (GF_CSC_PUSH_AG) — parity colocated + N=2/4 benches
P=gpurun_out/r2p
GF_CSC_PUSH_AG=1 timeout 600 python -m pytest tests/test_gpu_colocated.py -q -x -p no:cacheprovider -k "csc" > ${P}_colo.txt 2>&1
B="--steps 30 --warmup 5 --no-csc --no-e2e --no-cpu-baseline --trace"
for N in 4 2; do
  TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2962$N"
  for wl in resnet50-csc alexnet-csc; do
    for pag in 1 0; do
      GF_CSC_PUSH_AG=$pag timeout 200 $TR bench.py --gpus $N $B --workload $wl --csc-mode pull > ${P}_n${N}_${wl}_pag$pag.txt 2>&1
    done
    timeout 200 $TR bench.py --gpus $N $B --workload $wl --csc-mode push > ${P}_n${N}_${wl}_ring.txt 2>&1
  done
done

#!/bin/bash
# ncu on ONE rank of an N-process bench (the others run unprofiled): a single launch of the
# kernels matching $KREGEX is captured with --set full. The NVLink kernels' device-side
# barriers carry timeouts, so a peer waiting while the profiled rank replays cannot hang.
# usage: ncu_rank0.sh N KREGEX OUT.ncu-rep [bench args...]
N=$1; KRE=$2; OUT=$3; shift 3
export MASTER_ADDR=127.0.0.1 MASTER_PORT=29533 WORLD_SIZE=$N
pids=()
for r in $(seq 1 $((N-1))); do
  RANK=$r LOCAL_RANK=$r timeout 240 python bench.py --gpus $N "$@" > /dev/null 2>&1 &
  pids+=($!)
done
RANK=0 LOCAL_RANK=0 timeout 240 /usr/local/cuda/bin/ncu --set full --import-source on --clock-control none \
  -k "regex:$KRE" --launch-skip 6 --launch-count 1 -f -o $OUT python bench.py --gpus $N "$@" > ${OUT%.ncu-rep}.log 2>&1
for p in "${pids[@]}"; do wait $p; done

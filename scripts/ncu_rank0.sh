#!/bin/bash
# ncu on ONE rank of an N-process bench (the others run unprofiled): the launches matching
# KREGEX (skip S, count C) are captured with --set full. Only for kernels WITHOUT cross-rank
# waits (replays re-run them while the peers proceed). usage:
#   ncu_rank0.sh N KREGEX SKIP COUNT OUT.ncu-rep [bench args...]
N=$1; KRE=$2; SKIP=$3; CNT=$4; OUT=$5; shift 5
export MASTER_ADDR=127.0.0.1 MASTER_PORT=29533 WORLD_SIZE=$N
pids=()
for r in $(seq 1 $((N-1))); do
  RANK=$r LOCAL_RANK=$r timeout 300 python bench.py --gpus $N "$@" > ${OUT%.ncu-rep}_rank$r.log 2>&1 &
  pids+=($!)
done
RANK=0 LOCAL_RANK=0 timeout 300 /usr/local/cuda/bin/ncu --set full --import-source on --clock-control none \
  -k "regex:$KRE" --launch-skip $SKIP --launch-count $CNT -f -o $OUT python bench.py --gpus $N "$@" > ${OUT%.ncu-rep}.log 2>&1
for p in "${pids[@]}"; do wait $p; done

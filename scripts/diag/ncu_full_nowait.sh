#!/bin/bash
# ncu --set full of one launch of a multi-GPU kernel (one process drives N GPUs, GF_DIAG_NOWAIT=1:
# no waits, so the replayed kernel is its own work). usage: ncu_full_nowait.sh OUT N WORKLOAD MODE KREGEX
OUT=$1; N=$2; WL=$3; MODE=$4; KRE=$5
export GF_DIAG_NOWAIT=1 WORLD_SIZE=$N
STEPS=6 MODE=$MODE WORKLOAD=$WL timeout 400 /usr/local/cuda/bin/ncu --set full --import-source on --clock-control none \
  --devices 0 -k "regex:$KRE" -s 2 -c 1 -f -o $OUT python -u scripts/ncu_nvlink.py > $OUT.log 2>&1
echo "$OUT rc=$?"

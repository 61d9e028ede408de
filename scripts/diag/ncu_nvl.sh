#!/bin/bash
# ncu NVLink counters of the multi-GPU kernels: one process drives N GPUs, GF_DIAG_NOWAIT=1,
# rank 0's (device 0's) launches profiled. usage: ncu_nvl.sh OUTPREFIX N "workloads" "modes"
P=${1:-gpurun_out/nvl}; N=${2:-2}; WLS=${3:-"resnet50-dense alexnet-dense"}; MODES=${4:-"rspush pull push csc-push csc-pull"}
M=gpu__time_duration.sum,nvltx__bytes.sum,nvlrx__bytes.sum,nvltx__bytes_data_user.sum,nvlrx__bytes_data_user.sum,dram__bytes_read.sum,dram__bytes_write.sum
export GF_DIAG_NOWAIT=1 WORLD_SIZE=$N
for wl in $WLS; do
  for mode in $MODES; do
    STEPS=8 MODE=$mode WORKLOAD=$wl timeout 300 /usr/local/cuda/bin/ncu --metrics $M --clock-control none --devices 0 \
      -k 'regex:pack_push|rsp_kernel|rsag|ring_kernel|csc_pull|select_kernel|pack_correct|unpack_kernel|pack_kernel' \
      -s 4 -c 40 --csv --log-file ${P}_${wl}_${mode}.csv python -u scripts/ncu_nvlink.py > ${P}_${wl}_${mode}.log 2>&1
    echo "$wl $mode rc=$?"
  done
done

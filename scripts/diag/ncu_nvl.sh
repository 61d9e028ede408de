#!/bin/bash
# ncu NVLink counters of the multi-GPU kernels (rank 0 profiled, the others unprofiled, all with
# GF_DIAG_NOWAIT=1). usage: ncu_nvl.sh OUTPREFIX N "workloads" "modes"
P=${1:-gpurun_out/nvl}; N=${2:-2}; WLS=${3:-"resnet50-dense alexnet-dense"}; MODES=${4:-"rspush pull push csc-push csc-pull"}
M=gpu__time_duration.sum,nvltx__bytes.sum,nvlrx__bytes.sum,nvltx__bytes_data_user.sum,nvlrx__bytes_data_user.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed
export GF_DIAG_NOWAIT=1 WORLD_SIZE=$N
port=29561
for wl in $WLS; do
  for mode in $MODES; do
    port=$((port+1))
    for r in $(seq 1 $((N-1))); do
      PORT=$port MODE=$mode WORKLOAD=$wl RANK=$r timeout 300 python scripts/ncu_nvlink.py > ${P}_${wl}_${mode}_rank$r.log 2>&1 &
    done
    PORT=$port MODE=$mode WORKLOAD=$wl RANK=0 timeout 300 /usr/local/cuda/bin/ncu --metrics $M --clock-control none \
      -k 'regex:pack_push|rsp_kernel|rsag|ring_kernel|csc_pull|select_kernel|pack_correct|unpack_kernel|pack_kernel' \
      -s 8 -c 40 --csv --log-file ${P}_${wl}_${mode}.csv python scripts/ncu_nvlink.py > ${P}_${wl}_${mode}_rank0.log 2>&1
    echo "$wl $mode rc=$?"
    wait
  done
done

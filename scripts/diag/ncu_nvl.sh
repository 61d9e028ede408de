#!/bin/bash
P=${1:-gpurun_out/nvl}
M=gpu__time_duration.sum,nvltx__bytes.sum,nvlrx__bytes.sum,nvltx__bytes_data_user.sum,nvlrx__bytes_data_user.sum,dram__bytes_read.sum,dram__bytes_write.sum
for wl in resnet50-dense alexnet-dense; do
  WORKLOAD=$wl GF_PUSH_DIAG=2 RANK=1 timeout 200 python scripts/ncu_nvlink_pack.py > ${P}_${wl}_rank1.log 2>&1 &
  WORKLOAD=$wl GF_PUSH_DIAG=2 RANK=0 timeout 200 /usr/local/cuda/bin/ncu --metrics $M --clock-control none -k regex:pack_push -s 2 -c 3 --csv --log-file ${P}_${wl}.csv python scripts/ncu_nvlink_pack.py > ${P}_${wl}_rank0.log 2>&1
  wait
done

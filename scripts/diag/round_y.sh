#!/bin/bash
P=gpurun_out/r2y
bash scripts/diag/ncu_full_nowait.sh ${P}_rsp 2 resnet50-dense rspush rsp_kernel
bash scripts/diag/ncu_full_nowait.sh ${P}_packpush 2 resnet50-dense rspush pack_push
bash scripts/diag/ncu_full_nowait.sh ${P}_pipe 2 resnet50-dense pipe pipe_kernel
bash scripts/diag/ncu_nvl.sh ${P}_nvl4 4 "resnet50-dense" "rspush pipe" > ${P}_nvl4.txt 2>&1

#!/bin/bash
# 2-GPU box: rsp_kernel launch shapes (GF_RSP_CFG 0..5): parity colocated, N=2 step, NOWAIT ncu duration + NVLink
P=gpurun_out/r2z
for cfg in 3 4 5; do
  GF_RSP_CFG=$cfg timeout 300 python -m pytest tests/test_gpu_colocated.py -q -x -p no:cacheprovider -k "rspush or resnet50_full" > ${P}_colo_cfg$cfg.txt 2>&1
done
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29575"
B="--gpus 2 --steps 30 --warmup 5 --no-csc --no-e2e --no-cpu-baseline --trace"
for wl in resnet50-dense alexnet-dense; do
  for cfg in 0 1 2 3 4 5; do
    for fu in 1 0; do
      GF_FUSE_UNPACK=$fu GF_RSP_CFG=$cfg timeout 200 $TR bench.py $B --workload $wl --dense-mode rspush > ${P}_n2_${wl}_cfg${cfg}_fu${fu}.txt 2>&1
    done
  done
done
M=gpu__time_duration.sum,nvltx__bytes.sum,nvltx__bytes_data_user.sum,dram__bytes_read.sum,dram__bytes_write.sum
for cfg in 0 1 2 3 4 5; do
  GF_RSP_CFG=$cfg GF_DIAG_NOWAIT=1 WORLD_SIZE=2 STEPS=8 MODE=rspush WORKLOAD=resnet50-dense timeout 300 /usr/local/cuda/bin/ncu --metrics $M \
    --clock-control none --devices 0 -k regex:rsp_kernel -s 3 -c 3 --csv --log-file ${P}_nvl_cfg$cfg.csv python -u scripts/ncu_nvlink.py > ${P}_nvl_cfg$cfg.log 2>&1
done

#!/bin/bash
P=gpurun_out/r2o
bash scripts/diag/nvlink_smi_probe.sh > ${P}_nvsmi.txt 2>&1
timeout 900 python -m pytest tests/test_reference_suites.py tests/test_gpu_colocated.py tests/test_gflowpy.py -q -p no:cacheprovider -x > ${P}_tests.txt 2>&1
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29518"
timeout 300 $TR bench.py --gpus 2 --steps 30 --warmup 5 --no-e2e --workload alexnet-csc > ${P}_n2_acsc.txt 2>&1
timeout 300 $TR bench.py --gpus 2 --steps 30 --warmup 5 --no-e2e --workload resnet50-csc > ${P}_n2_rcsc.txt 2>&1
timeout 300 python bench.py --steps 20 --warmup 5 > ${P}_bench1.txt 2>&1

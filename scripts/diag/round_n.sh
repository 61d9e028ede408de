#!/bin/bash
P=gpurun_out/r2n
timeout 600 python -m pytest tests/test_reference_suites.py tests/test_gpu_stress.py -q -p no:cacheprovider -k "reference or colocated" > ${P}_tests.txt 2>&1
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517"
timeout 300 $TR bench.py --gpus 2 --steps 30 --warmup 5 --no-e2e --workload alexnet-csc > ${P}_n2_acsc.txt 2>&1
timeout 300 $TR bench.py --gpus 2 --steps 30 --warmup 5 --no-e2e --workload resnet50-csc > ${P}_n2_rcsc.txt 2>&1
bash scripts/ncu_rank0.sh 2 pack_correct 6 2 ${P}_pc.ncu-rep --workload alexnet-csc --steps 6 --warmup 3 --no-e2e --no-cpu-baseline
timeout 300 $TR scripts/nvlink_counters.py --steps 100 > ${P}_nvcount.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_stress.py -q -p no:cacheprovider -k multigpu > ${P}_stress_multi.txt 2>&1

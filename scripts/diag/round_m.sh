#!/bin/bash
P=gpurun_out/r2m
timeout 900 python -m pytest tests/test_gflowpy.py tests/test_reference_suites.py tests/test_gpu_colocated.py tests/test_gpu_kernels.py -q -p no:cacheprovider > ${P}_tests.txt 2>&1
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29516"
timeout 300 $TR bench.py --gpus 2 --steps 30 --warmup 5 --no-e2e --trace > ${P}_n2_resnet.txt 2>&1
timeout 300 $TR bench.py --gpus 2 --steps 30 --warmup 5 --no-e2e --no-csc --workload alexnet-dense --trace > ${P}_n2_alexnet.txt 2>&1
timeout 300 $TR bench.py --gpus 2 --steps 30 --warmup 5 --no-e2e --workload resnet50-csc > ${P}_n2_rcsc.txt 2>&1
timeout 300 python bench.py --steps 20 --warmup 5 > ${P}_bench1.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_multi.py -q -p no:cacheprovider > ${P}_multi.txt 2>&1

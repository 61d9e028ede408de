#!/bin/bash
# N-GPU bench sweep of the default dense path + CSC at N GPUs
N=${1:-4}; P=gpurun_out/r2p_n${N}
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29519"
timeout 300 $TR bench.py --gpus $N --steps 30 --warmup 5 --no-e2e --trace > ${P}_resnet.txt 2>&1
timeout 300 $TR bench.py --gpus $N --steps 30 --warmup 5 --no-e2e --no-csc --workload alexnet-dense --trace > ${P}_alexnet.txt 2>&1
timeout 300 $TR bench.py --gpus $N --steps 30 --warmup 5 --no-e2e --workload resnet50-csc > ${P}_rcsc.txt 2>&1
GF_CSC_XBLOCKS=32 timeout 300 $TR bench.py --gpus $N --steps 30 --warmup 5 --no-e2e --workload alexnet-csc > ${P}_acsc32.txt 2>&1
GF_PUSH_DIAG=1 timeout 300 $TR bench.py --gpus $N --steps 30 --warmup 5 --no-e2e --no-csc > ${P}_diag1.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_multi.py tests/test_gpu_stress.py -q -p no:cacheprovider -k "multigpu or p2p or tcp" > ${P}_multi.txt 2>&1

timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_multi.py -x -q -k "csc" > gpurun_out/pt.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pt.log
for w in alexnet-csc resnet50-csc; do for tma in 1 0; do
  GF_PACK_CORRECT_TMA=$tma CUDA_VISIBLE_DEVICES=0 timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --workload $w > gpurun_out/tma${tma}_$w.log 2>&1
  grep "^{" gpurun_out/tma${tma}_$w.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w tma=$tma', d['value'], json.dumps(d['kernels']))"
done; done
GF_PACK_CORRECT_TMA=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 30 --warmup 5 --no-e2e --no-cpu-baseline --workload alexnet-csc > gpurun_out/tma1_n2.log 2>&1
grep "^{" gpurun_out/tma1_n2.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('N2 alexnet-csc tma=1', d['value'], json.dumps(d['kernels']))"

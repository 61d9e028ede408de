timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q -k "sgd or csc" > gpurun_out/pt.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pt.log
for w in alexnet-csc resnet50-csc; do
  CUDA_VISIBLE_DEVICES=0 timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --workload $w > gpurun_out/sgd_$w.log 2>&1
  grep "^{" gpurun_out/sgd_$w.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w', d['value'], json.dumps(d['kernels']))"
done
NCCL_DEBUG=INFO NCCL_DEBUG_SUBSYS=INIT,NVLS timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 scripts/nvls_probe.py > gpurun_out/nvls_probe.log 2>&1; echo "nvls rc=$?"
grep -E "NVLS|multicast|bytes=" gpurun_out/nvls_probe.log | grep -v "^\s*$" | head -12

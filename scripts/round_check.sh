# One gpurun call: GPU parity suite, N=1 bench of every workload, N=2 bench, NVLS probe.
set -x
mkdir -p gpurun_out
nvidia-smi topo -m > gpurun_out/topo.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
for w in resnet50-dense alexnet-dense alexnet-csc resnet50-csc; do
  timeout 600 python bench.py --steps 20 --warmup 5 --workload $w > gpurun_out/bench_n1_$w.log 2>&1; echo "bench $w rc=$?"
  grep '^{' gpurun_out/bench_n1_$w.log | tail -1 | cut -c1-400
done
NG=$(nvidia-smi -L | wc -l)
if [ "$NG" -ge 2 ]; then
  for w in resnet50-dense alexnet-dense alexnet-csc; do
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $NG --steps 20 --warmup 5 --workload $w --no-e2e > gpurun_out/bench_n${NG}_$w.log 2>&1; echo "bench N=$NG $w rc=$?"
    grep '^{' gpurun_out/bench_n${NG}_$w.log | tail -1 | cut -c1-400
  done
  NCCL_DEBUG=INFO NCCL_DEBUG_SUBSYS=INIT,NVLS timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29512 scripts/nvls_probe.py > gpurun_out/nvls_probe.log 2>&1; echo "nvls rc=$?"
  grep -E "NVLS|multicast" gpurun_out/nvls_probe.log | grep -v "^\s*$" | head -20
fi

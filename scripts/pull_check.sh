# dense pull-mode check: multi-GPU parity of the new path, then N=all benches pull vs push
mkdir -p gpurun_out
NG=$(nvidia-smi -L | wc -l)
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -k "unpack or fused_step or ring_bit" > gpurun_out/pytest_pull.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_pull.log
for w in resnet50-dense alexnet-dense; do
  for m in pull push; do
    timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $NG --steps 30 --warmup 5 --workload $w --no-e2e --no-cpu-baseline --dense-mode $m ${TRACE:+--trace} > gpurun_out/bench_${m}_n${NG}_$w.log 2>&1; echo "bench $m N=$NG $w rc=$?"
    grep '^{' gpurun_out/bench_${m}_n${NG}_$w.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['bus_gbs'], json.dumps(d['kernels']), d.get('ring_trace'))"
  done
done

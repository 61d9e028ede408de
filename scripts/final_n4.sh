mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pt4.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pt4.log
NG=$(nvidia-smi -L | wc -l)
run() {
  timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $NG --steps 30 --warmup 5 $2 > gpurun_out/fin_$1_n$NG.log 2>&1
  echo "== $1 N=$NG rc=$?"
  grep '^{' gpurun_out/fin_$1_n$NG.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['config'].get('exchange'), d['bus_gbs'], json.dumps(d['kernels']), 'e2e', (d.get('e2e') or {}).get('value'), 'nccl', d.get('nccl_allreduce'))" 2>&1 | tail -1
}
run rdef ""
run adef "--workload alexnet-dense --no-e2e"
run cdef "--workload alexnet-csc --no-e2e"
run rcsc "--workload resnet50-csc --no-e2e"

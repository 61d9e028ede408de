# N = all GPUs of the box: default benches (with e2e) in every mode, plus the NCCL comparison
mkdir -p gpurun_out
NG=$(nvidia-smi -L | wc -l)
run() {  # label, args
  timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $NG --steps 30 --warmup 5 $2 > gpurun_out/sc_$1_n$NG.log 2>&1
  echo "== $1 N=$NG rc=$?"
  grep '^{' gpurun_out/sc_$1_n$NG.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['bus_gbs'], json.dumps(d['kernels']), 'e2e', (d.get('e2e') or {}).get('value'), 'nccl', d.get('nccl_allreduce'), 'launches', d.get('gpu_launches'))" 2>&1 | tail -1
}
run rpull "--workload resnet50-dense"
run rpush "--workload resnet50-dense --dense-mode push"
run rfused "--workload resnet50-dense --dense-mode fused --no-e2e"
run apull "--workload alexnet-dense"
run apush "--workload alexnet-dense --dense-mode push --no-e2e"
run cpull "--workload alexnet-csc"
run cpush "--workload alexnet-csc --csc-mode push --no-e2e"
run r5csc "--workload resnet50-csc --no-e2e"

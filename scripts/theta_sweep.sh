NG=$(nvidia-smi -L | wc -l)
for th in 0 262144 1048576 4194304 -1; do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $NG --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --workload resnet50-csc --theta $th $CSCARGS > gpurun_out/theta_${th}_n$NG.log 2>&1
  grep '^{' gpurun_out/theta_${th}_n$NG.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('theta', $th, d['value'], json.dumps(d['kernels']))"
done

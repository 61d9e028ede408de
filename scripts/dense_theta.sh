NG=$(nvidia-smi -L | wc -l)
for mode in push pull; do
for th in 0 1048576 4194304 -1; do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $NG --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --workload resnet50-dense --theta $th --dense-mode $mode > gpurun_out/dtheta_${mode}_${th}_n$NG.log 2>&1
  grep '^{' gpurun_out/dtheta_${mode}_${th}_n$NG.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$mode theta', $th, d['value'], json.dumps(d['kernels']))"
done; done
for w in resnet50-dense alexnet-dense; do for mode in push pull; do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $NG --steps 30 --warmup 5 --no-e2e --no-cpu-baseline --workload $w --dense-mode $mode > gpurun_out/d_${mode}_${w}_n$NG.log 2>&1
  grep '^{' gpurun_out/d_${mode}_${w}_n$NG.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w $mode', d['value'], json.dumps(d['kernels']))"
done; done

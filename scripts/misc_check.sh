NG=$(nvidia-smi -L | wc -l)
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $NG --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --overlap 2 > gpurun_out/ov_n$NG.log 2>&1; echo "overlap rc=$?"
grep '^{' gpurun_out/ov_n$NG.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d.get('overlap'))"
timeout 400 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --overlap 2 > gpurun_out/ov_n1.log 2>&1; echo "overlap n1 rc=$?"
grep '^{' gpurun_out/ov_n1.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d.get('overlap'))"
for m in push pull; do
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $NG --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --workload resnet50-csc --theta 0 --csc-mode $m > gpurun_out/csc0_$m.log 2>&1; echo "csc theta0 $m rc=$?"
grep '^{' gpurun_out/csc0_$m.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], json.dumps(d['kernels']))"
done

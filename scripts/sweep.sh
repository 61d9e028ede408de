# usage: bash scripts/sweep.sh "<label>|<bench args>" ...   (runs each at N = all GPUs of the box)
mkdir -p gpurun_out
NG=$(nvidia-smi -L | wc -l)
for spec in "$@"; do
  label=${spec%%|*}; bargs=${spec#*|}
  if [ "$NG" -gt 1 ]; then
    timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $NG --steps 30 --warmup 5 --no-e2e --no-cpu-baseline $bargs > gpurun_out/sw_${label}_n$NG.log 2>&1
  else
    timeout 300 python bench.py --steps 30 --warmup 5 --no-e2e --no-cpu-baseline $bargs > gpurun_out/sw_${label}_n$NG.log 2>&1
  fi
  echo "== $label N=$NG rc=$?"
  grep '^{' gpurun_out/sw_${label}_n$NG.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['bus_gbs'], json.dumps(d['kernels']), d.get('ring_trace'))" 2>&1 | tail -1
done

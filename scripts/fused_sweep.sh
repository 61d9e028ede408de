# Sweep the NVLink-CTA count of the fused step. Usage: fused_sweep.sh N "R1 R2 ..." [bench args]
N=$1; RS=$2; shift 2
for R in $RS; do
  echo "== GF_STEP_RED=$R"
  GF_STEP_RED=$R timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N \
    --master-addr 127.0.0.1 --master-port $((29600 + R)) bench.py --gpus $N --fused --no-e2e "$@" 2>&1 \
    | grep '^{' | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['kernels'], d.get('nccl_allreduce'))"
done

# usage: bash scripts/bench_multi.sh "2 4" [extra bench args]
NS=${1:-"2 4"}; shift
for n in $NS; do
  python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $n "$@" 2>&1 | grep '^{' ;
done

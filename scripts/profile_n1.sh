# ncu evidence for N=1 bench workloads (B200_PROFILING.md recipe). Usage: profile_n1.sh TAG
TAG=${1:-r1}
run() {  # $1 workload  $2 kernel regex
  W=$1; CMD="python bench.py --steps 6 --warmup 3 --no-cpu-baseline --no-e2e --no-csc --workload $W"
  $CMD > gpurun_out/plain_$W.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches_${W}_$TAG.csv $CMD > gpurun_out/ncu_launch_$W.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"$2" -s 8 -c 8 -o gpurun_out/prof_${W}_$TAG $CMD > gpurun_out/ncu_full_$W.log 2>&1
  echo "$W rc=$?"
}
run resnet50-dense "pack_kernel|unpack_kernel"
run alexnet-dense "pack_kernel|unpack_kernel"
run alexnet-csc "pack_correct|select_kernel|compact_kernel|csc_sgd"

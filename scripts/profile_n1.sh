# ncu evidence for N=1 bench workloads (B200_PROFILING.md recipe). Usage: profile_n1.sh TAG
# Summaries are written on the box (scripts/ncu_summary.py, scripts/ncu_traffic.py); the
# --set full reports are kept only for the first workload (gpurun_out is capped at 64 MiB).
TAG=${1:-r1}
reps=()
run() {  # $1 workload  $2 kernel regex
  W=$1; CMD="python bench.py --steps 6 --warmup 3 --no-cpu-baseline --no-e2e --no-csc --workload $W"
  $CMD > gpurun_out/plain_$W.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches_${W}_$TAG.csv $CMD > gpurun_out/ncu_launch_$W.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"$2" -s 8 -c 2 -f -o gpurun_out/prof_${W}_$TAG $CMD > gpurun_out/ncu_full_$W.log 2>&1
  echo "$W rc=$?"
  python scripts/ncu_summary.py gpurun_out/launches_${W}_$TAG.csv gpurun_out/prof_${W}_$TAG.ncu-rep > gpurun_out/${TAG}f_${W//-/_}_n1.md 2>&1
  reps+=("$W=gpurun_out/prof_${W}_$TAG.ncu-rep")
}
run resnet50-dense "pack_kernel|unpack_kernel"
run alexnet-dense "pack_kernel|unpack_kernel"
run alexnet-csc "pack_correct|select_kernel|compact_kernel|csc_sgd"
python scripts/ncu_traffic.py $TAG "${reps[@]}" > gpurun_out/ncu_traffic_$TAG.json 2>&1
rm -f gpurun_out/prof_alexnet-dense_$TAG.ncu-rep gpurun_out/prof_alexnet-csc_$TAG.ncu-rep
du -sh gpurun_out

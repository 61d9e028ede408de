# ncu evidence for the N=1 default bench (see B200_PROFILING.md). Args: workload tag
W=${1:-resnet50-dense}; TAG=${2:-r1}
CMD="python bench.py --steps 6 --warmup 3 --no-cpu-baseline --no-e2e --workload $W"
$CMD > gpurun_out/plain_$W.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches_${W}_$TAG.csv $CMD > gpurun_out/ncu_launch_$W.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"${3:-pack_kernel|unpack_kernel}" -s 4 -c 4 -o gpurun_out/prof_${W}_$TAG $CMD > gpurun_out/ncu_full_$W.log 2>&1
echo "rc=$?"

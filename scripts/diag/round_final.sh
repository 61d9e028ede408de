#!/bin/bash
# Round-2 evidence on a 4-GPU box: full GPU suite, smoke, N=1 bench (+ reference arm), N=2/4 benches
# of every workload, ncu of the N=1 kernels, NVLink ncu of the N=4 kernels.
P=gpurun_out/r2f
nvidia-smi -L > ${P}_gpus.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > ${P}_pytest.txt 2>&1; echo "pytest rc=$?" >> ${P}_pytest.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > ${P}_smoke.txt 2>&1
timeout 600 python bench.py > ${P}_bench_n1.txt 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > ${P}_bench_ref_n1.txt 2>&1
for w in alexnet-dense resnet50-csc; do
  timeout 400 python bench.py --steps 20 --warmup 5 --workload $w --no-e2e --no-csc > ${P}_bench_n1_$w.txt 2>&1
done
for N in 2 4; do
  TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2958$N"
  timeout 600 $TR bench.py --gpus $N --trace > ${P}_bench_n${N}.txt 2>&1
  for w in alexnet-dense resnet50-csc alexnet-csc; do
    timeout 400 $TR bench.py --gpus $N --steps 30 --warmup 5 --workload $w --no-csc --no-e2e --no-cpu-baseline --trace > ${P}_bench_n${N}_$w.txt 2>&1
  done
done
bash scripts/profile_n1.sh r2 > ${P}_profile_n1.txt 2>&1
bash scripts/diag/ncu_nvl.sh ${P}_nvl4 4 "resnet50-dense alexnet-dense" "rspush push pull csc-push csc-pull" > ${P}_nvl4.txt 2>&1
bash scripts/diag/ncu_nvl.sh ${P}_nvl2 2 "alexnet-dense" "rspush csc-push" > ${P}_nvl2.txt 2>&1

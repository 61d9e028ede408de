#!/bin/bash
# evidence run on a 4-GPU box: full GPU suite, benches at N=1/2/4, ncu at N=1, NVLink ncu of the routed pack
P=gpurun_out/r2s
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > ${P}_pytest.txt 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > ${P}_smoke.txt 2>&1
timeout 400 python bench.py > ${P}_bench_n1.txt 2>&1
timeout 400 python bench.py --impl reference --steps 3 --warmup 1 > ${P}_bench_ref_n1.txt 2>&1
for N in 2 4; do
  TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2955$N"
  timeout 600 $TR bench.py --gpus $N --trace > ${P}_bench_n${N}.txt 2>&1
  timeout 400 $TR bench.py --gpus $N --steps 30 --warmup 5 --workload alexnet-dense --no-csc --trace > ${P}_bench_n${N}_alexnet.txt 2>&1
done
bash scripts/profile_n1.sh r2 > ${P}_profile_n1.txt 2>&1
bash scripts/diag/ncu_nvl.sh ${P}_nvl > ${P}_nvl.txt 2>&1

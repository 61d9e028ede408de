#!/bin/bash
# 1-GPU evidence (what the driver runs): GPU suite, smoke, N=1 benches (+ reference arm), ncu
P=gpurun_out/r2f1
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > ${P}_pytest.txt 2>&1; echo "pytest rc=$?" >> ${P}_pytest.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > ${P}_smoke.txt 2>&1
timeout 600 python bench.py > ${P}_bench_n1.txt 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > ${P}_bench_ref_n1.txt 2>&1
for w in alexnet-dense resnet50-csc alexnet-csc; do
  timeout 400 python bench.py --steps 20 --warmup 5 --workload $w --no-e2e --no-csc > ${P}_bench_n1_$w.txt 2>&1
done
bash scripts/profile_n1.sh r2 > ${P}_profile_n1.txt 2>&1

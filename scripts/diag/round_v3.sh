#!/bin/bash
# 1-GPU final verification (what the driver runs)
P=gpurun_out/r2v3
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > ${P}_pytest.txt 2>&1; echo "pytest rc=$?" >> ${P}_pytest.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > ${P}_smoke.txt 2>&1
timeout 600 python bench.py > ${P}_bench_n1.txt 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > ${P}_bench_ref_n1.txt 2>&1
timeout 400 python bench.py --steps 20 --warmup 5 --workload resnet50-csc --no-e2e --no-csc > ${P}_bench_n1_resnet50-csc.txt 2>&1

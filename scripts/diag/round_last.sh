#!/bin/bash
# last sanity (1 GPU): the update tests and the gflowpy trainer after the compile-time-only edit
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gflowpy.py -m gpu -q -p no:cacheprovider -k "sgd or train or rooted" > gpurun_out/r2last_pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/r2last_pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2last_smoke.txt 2>&1

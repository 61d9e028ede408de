#!/bin/bash
# 1-GPU: rooted collectives (pointers in parameter space, 16-byte vectors) and the vectorised dense
# momentum update: the reference's suites, gflowpy's rooted/train goldens, the update tests
P=gpurun_out/r2rt
timeout 900 python -m pytest tests/test_reference_suites.py tests/test_gflowpy.py tests/test_gpu_kernels.py -m gpu -q -p no:cacheprovider > ${P}_pytest.txt 2>&1; echo "rc=$?" >> ${P}_pytest.txt

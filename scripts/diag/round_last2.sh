#!/bin/bash
timeout 600 python -m pytest tests/test_gpu_colocated.py -q -p no:cacheprovider -k "csc" > gpurun_out/r2last2_colo_csc.txt 2>&1; echo "rc=$?" >> gpurun_out/r2last2_colo_csc.txt

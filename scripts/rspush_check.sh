timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -k "fused_step" > gpurun_out/pt.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pt.log
bash scripts/sweep.sh "rsp|--workload resnet50-dense --dense-mode rspush --trace" "rpl|--workload resnet50-dense --dense-mode pull" "asp|--workload alexnet-dense --dense-mode rspush" "apl|--workload alexnet-dense --dense-mode pull" "rsp0|--workload resnet50-dense --dense-mode rspush --theta 0"
bash scripts/misc_check.sh

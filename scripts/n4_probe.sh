mkdir -p gpurun_out
NG=$(nvidia-smi -L | wc -l)
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29517 scripts/ce_probe.py > gpurun_out/ce_probe_n$NG.log 2>&1; echo "ce rc=$?"; grep "^N=" gpurun_out/ce_probe_n$NG.log
bash scripts/config45.sh

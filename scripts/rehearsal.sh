# round-end rehearsal: smoke, default bench (N=1), reference arm, N=2 both arms
mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/reh_n1.log 2>&1; echo "bench rc=$?"; grep '^{' gpurun_out/reh_n1.log | cut -c1-300
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/reh_ref_n1.log 2>&1; echo "ref rc=$?"; grep '^{' gpurun_out/reh_ref_n1.log | cut -c1-400
NG=$(nvidia-smi -L | wc -l)
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29521 bench.py --gpus $NG > gpurun_out/reh_n$NG.log 2>&1; echo "bench N=$NG rc=$?"; grep '^{' gpurun_out/reh_n$NG.log | cut -c1-300
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29522 bench.py --gpus $NG --impl reference --steps 3 --warmup 3 > gpurun_out/reh_ref_n$NG.log 2>&1; echo "ref N=$NG rc=$?"; grep '^{' gpurun_out/reh_ref_n$NG.log | cut -c1-400

# SPDX-License-Identifier: Apache-2.0
"""NVLink hardware counters per launch of the NVLink kernels (torchrun, one process per GPU).

NVML's cumulative per-link NVLink throughput counters (NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX/RX
and _RAW_TX/RX, KiB, summed over the GPU's links) are read on every rank before and after K
back-to-back launches of one piece of the path, with CUDA-event device time around them:

  rspush_step   the default dense step (routed pack + rsp_kernel with the fused unpack);
                run with GF_PUSH_DIAG=2 it is the routed pack alone (results invalid)
  csc_step      the CSC step (pack_correct + exchange + select + update), AlexNet
  nccl          torch.distributed.all_reduce of the same fp16 pool bytes (comparison)

Prints one JSON line per piece (rank 0): bytes per launch per GPU (max over ranks), the
algorithmic bytes that piece must move, and the achieved GB/s of the counted bytes.
    torchrun --nproc-per-node N scripts/nvlink_counters.py [--steps K] [--workload W]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def nvlink_kib(nv, h):
    fids = [nv.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX, nv.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_RX,
            nv.NVML_FI_DEV_NVLINK_THROUGHPUT_RAW_TX, nv.NVML_FI_DEV_NVLINK_THROUGHPUT_RAW_RX]
    tot = [0, 0, 0, 0]
    for link in range(18):
        try:
            vals = nv.nvmlDeviceGetFieldValues(h, [(f, link) for f in fids])
        except Exception:
            break
        for i, v in enumerate(vals):
            if v.nvmlReturn == 0:
                tot[i] += int(v.value.ullVal)
    return tot


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--workload", default="resnet50-dense")
    args = ap.parse_args()
    import numpy as np
    import pynvml as nv
    import torch
    import torch.distributed as dist
    import bench
    from paper_1902_06855_b200 import capi, cudart
    from paper_1902_06855_b200.engine import GradSync
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    cudart.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    nv.nvmlInit()
    h = nv.nvmlDeviceGetHandleByIndex(local)

    def ag(b):
        out = [None] * world
        dist.all_gather_object(out, b)
        return out

    stream = torch.cuda.current_stream()
    sp = stream.cuda_stream
    results = []

    def measure(name, step, algo_bytes):
        for i in range(5):
            step(i)
        torch.cuda.synchronize()
        dist.barrier()
        c0 = nvlink_kib(nv, h)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for i in range(args.steps):
            step(i)
        e1.record(stream)
        torch.cuda.synchronize()
        dist.barrier()
        c1 = nvlink_kib(nv, h)
        per = [(b - a) * 1024 / args.steps for a, b in zip(c0, c1)]
        ms = e0.elapsed_time(e1) / args.steps
        t = torch.tensor(per + [ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        per, ms = t[:4].tolist(), float(t[4])
        results.append({"piece": name, "n_gpus": world, "ms_per_launch": round(ms, 4),
                        "nvlink_data_tx_bytes": int(per[0]), "nvlink_data_rx_bytes": int(per[1]),
                        "nvlink_raw_tx_bytes": int(per[2]), "nvlink_raw_rx_bytes": int(per[3]),
                        "algorithmic_bytes_per_direction": int(algo_bytes),
                        "data_tx_GBps": round(per[0] / (ms / 1e3) / 1e9, 1),
                        "data_vs_algorithmic": round(per[0] / algo_bytes, 4) if algo_bytes else None})

    wl = bench.WORKLOADS[args.workload]
    sizes = wl["sizes"]
    total = sum(sizes)
    bounds = np.concatenate([[0], np.cumsum(sizes)])
    import ctypes as C
    sets = [torch.from_numpy(capi.synth_grads(rank, t, sizes)).cuda() for t in range(2)]
    out = torch.empty(total, device="cuda")

    def table(flat):
        return (C.c_void_p * len(sizes))(*[flat[int(bounds[i]):int(bounds[i + 1])].data_ptr() for i in range(len(sizes))])

    gt = [table(x) for x in sets]
    ot = table(out)
    K = total * 2  # fp16 pool bytes
    eng = GradSync(sizes, rank=rank, world=world, device=local, theta=wl["theta"], allgather=ag)
    measure("rspush_step", lambda i: eng.dense_step(gt[i % 2], ot, stream=sp), 2 * (world - 1) * K // world)
    eng.close()
    x = torch.zeros(total, dtype=torch.float16, device="cuda")
    measure("nccl_allreduce", lambda i: dist.all_reduce(x), 2 * (world - 1) * K // world)
    csc = bench.WORKLOADS["alexnet-csc"]
    ceng = GradSync(csc["sizes"], rank=rank, world=world, device=local, theta=csc["theta"], csc=True,
                    final_sparsity=0.9, allgather=ag)
    ctotal = sum(csc["sizes"])
    cb = np.concatenate([[0], np.cumsum(csc["sizes"])])
    cset = torch.from_numpy(capi.synth_grads(rank, 0, csc["sizes"])).cuda()
    ct = (C.c_void_p * len(csc["sizes"]))(*[cset[int(cb[i]):int(cb[i + 1])].data_ptr() for i in range(len(csc["sizes"]))])
    for i in range(3):  # past the dense iteration 0
        ceng.csc_step(ct, stream=sp)
    k = 191 * 32000 * 2
    measure("csc_step_alexnet", lambda i: ceng.csc_step(ct, stream=sp), 2 * (world - 1) * k // world)
    ceng.close()
    if rank == 0:
        for r in results:
            print(json.dumps(r), flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()

# SPDX-License-Identifier: Apache-2.0
"""NVLink bytes per launch of the routed pack, from ncu's nvltx/nvlrx counters.

Two processes (gloo bootstrap, no NCCL), one per GPU. Both run the engine's rspush step with
GF_PUSH_DIAG=2 — the routed pack alone, no cross-rank wait anywhere (results invalid by design) —
so rank 0 can run under ncu (kernel replay re-issues the NVLink stores into rank 1's inbox:
idempotent) while rank 1 runs unprofiled. Usage (repo root, 2 GPUs):
    bash -c 'GF_PUSH_DIAG=2 RANK=1 python scripts/ncu_nvlink_pack.py & \\
             GF_PUSH_DIAG=2 RANK=0 ncu --metrics <list> -k regex:pack_push python scripts/ncu_nvlink_pack.py'
"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_1902_06855_b200 import capi, cudart
    from paper_1902_06855_b200.engine import GradSync
    import bench
    rank, world = int(os.environ["RANK"]), int(os.environ.get("WORLD_SIZE", 2))
    torch.cuda.set_device(rank)
    cudart.set_device(rank)
    dist.init_process_group("gloo", init_method="tcp://127.0.0.1:29541", rank=rank, world_size=world)

    def ag(b):
        out = [None] * world
        dist.all_gather_object(out, b)
        return out

    wl = bench.WORKLOADS[os.environ.get("WORKLOAD", "resnet50-dense")]
    sizes = wl["sizes"]
    g = torch.from_numpy(capi.synth_grads(rank, 0, sizes)).cuda()
    out = torch.empty_like(g)
    b = np.concatenate([[0], np.cumsum(sizes)])
    gt = (C.c_void_p * len(sizes))(*[g[int(b[i]):int(b[i + 1])].data_ptr() for i in range(len(sizes))])
    ot = (C.c_void_p * len(sizes))(*[out[int(b[i]):int(b[i + 1])].data_ptr() for i in range(len(sizes))])
    eng = GradSync(sizes, rank=rank, world=world, device=rank, theta=wl["theta"], allgather=ag)
    for _ in range(int(os.environ.get("STEPS", 6))):
        eng.dense_step(gt, ot)
    torch.cuda.synchronize()
    dist.barrier()
    eng.close()
    if rank == 0:
        print("total elements", sum(sizes), "fp16 pool bytes", 2 * sum(sizes),
              "expected NVLink TX per launch (N-1)/N*K =", (world - 1) * 2 * sum(sizes) // world)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()

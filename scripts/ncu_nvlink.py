# SPDX-License-Identifier: Apache-2.0
"""NVLink bytes per launch of the multi-GPU kernels, from ncu's nvltx/nvlrx counters.

N processes (gloo bootstrap, no NCCL), one per GPU, each running the engine's step for MODE
(rspush | pull | push | csc-push | csc-pull) on WORKLOAD's seeded gradients. Run with
GF_DIAG_NOWAIT=1: the cross-GPU barriers signal but never wait, so rank 0 can run under ncu
(kernel replay re-issues the same stores into the peers' buffers) while the other ranks run
unprofiled. Every result is invalid by design; only the traffic and the kernel durations
without waits are measured. scripts/diag/ncu_nvl.sh drives it.
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
    assert os.environ.get("GF_DIAG_NOWAIT") == "1", "a traffic probe: run with GF_DIAG_NOWAIT=1"
    rank, world = int(os.environ["RANK"]), int(os.environ.get("WORLD_SIZE", 2))
    torch.cuda.set_device(rank)
    cudart.set_device(rank)
    dist.init_process_group("gloo", init_method="tcp://127.0.0.1:%s" % os.environ.get("PORT", "29541"),
                            rank=rank, world_size=world)

    def ag(b):
        out = [None] * world
        dist.all_gather_object(out, b)
        return out

    mode = os.environ.get("MODE", "rspush")
    wl = bench.WORKLOADS[os.environ.get("WORKLOAD", "resnet50-dense")]
    sizes = wl["sizes"]
    g = torch.from_numpy(capi.synth_grads(rank, 0, sizes)).cuda()
    out = torch.empty_like(g)
    b = np.concatenate([[0], np.cumsum(sizes)])
    gt = (C.c_void_p * len(sizes))(*[g[int(b[i]):int(b[i + 1])].data_ptr() for i in range(len(sizes))])
    ot = (C.c_void_p * len(sizes))(*[out[int(b[i]):int(b[i + 1])].data_ptr() for i in range(len(sizes))])
    if mode.startswith("csc"):
        eng = GradSync(sizes, rank=rank, world=world, device=rank, theta=wl["theta"], allgather=ag, csc=True,
                       csc_mode=mode.split("-")[1], final_sparsity=0.9)
        step = lambda: eng.csc_step(gt)  # noqa: E731
    else:
        eng = GradSync(sizes, rank=rank, world=world, device=rank, theta=wl["theta"], allgather=ag,
                       dense_mode=mode)
        step = lambda: eng.dense_step(gt, ot)  # noqa: E731
    for _ in range(int(os.environ.get("STEPS", 6))):
        step()
    torch.cuda.synchronize()
    dist.barrier()  # every rank keeps its (peer-mapped) heap until all are done
    eng.close()
    if rank == 0:
        K = 2 * sum(sizes)
        print("mode", mode, "elements", sum(sizes), "fp16 pool bytes", K,
              "ring NVLink bytes per direction 2(N-1)/N*K =", 2 * (world - 1) * K // world)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()

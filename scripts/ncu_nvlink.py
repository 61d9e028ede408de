# SPDX-License-Identifier: Apache-2.0
"""NVLink bytes per launch of the multi-GPU kernels, from ncu's nvltx/nvlrx counters.

ONE process drives N ranks on N GPUs (peer access, GradSync.local), each running the engine's
step for MODE (rspush | pull | push | csc-push | csc-pull) on WORKLOAD's seeded
gradients. Run with GF_DIAG_NOWAIT=1: the cross-GPU barriers and flags signal but never wait, so
ncu can serialise and replay each kernel (replays re-issue the same stores into the peers'
buffers). Every result is invalid by design; only the traffic and the kernel durations without
waits are measured. scripts/diag/ncu_nvl.sh drives it (ncu --devices 0: rank 0's launches).
"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import numpy as np
    import torch
    from paper_1902_06855_b200 import capi, cudart
    from paper_1902_06855_b200.engine import GradSync
    import bench
    assert os.environ.get("GF_DIAG_NOWAIT") == "1", "a traffic probe: run with GF_DIAG_NOWAIT=1"
    world = int(os.environ.get("WORLD_SIZE", 2))
    mode = os.environ.get("MODE", "rspush")
    wl = bench.WORKLOADS[os.environ.get("WORKLOAD", "resnet50-dense")]
    sizes = wl["sizes"]
    b = np.concatenate([[0], np.cumsum(sizes)])
    kw = dict(theta=wl["theta"])
    if mode.startswith("csc"):
        kw.update(csc=True, csc_mode=mode.split("-")[1], final_sparsity=0.9)
    else:
        kw.update(dense_mode=mode)
    ranks = GradSync.local(world, sizes, **kw)
    tabs = []
    for r in range(world):
        torch.cuda.set_device(r)
        g = torch.from_numpy(capi.synth_grads(r, 0, sizes)).cuda(r)
        out = torch.empty_like(g)
        gt = (C.c_void_p * len(sizes))(*[g[int(b[i]):int(b[i + 1])].data_ptr() for i in range(len(sizes))])
        ot = (C.c_void_p * len(sizes))(*[out[int(b[i]):int(b[i + 1])].data_ptr() for i in range(len(sizes))])
        tabs.append((g, out, gt, ot))
    for _ in range(int(os.environ.get("STEPS", 4))):
        for r in range(world):
            cudart.set_device(r)
            if mode.startswith("csc"):
                ranks[r].csc_step(tabs[r][2])
            else:
                ranks[r].dense_step(tabs[r][2], tabs[r][3])
    for r in range(world):
        torch.cuda.synchronize(r)
    for g in ranks:
        g.close()
    K = 2 * sum(sizes)
    print("mode", mode, "world", world, "elements", sum(sizes), "fp16 pool bytes", K,
          "ring NVLink bytes per direction 2(N-1)/N*K =", 2 * (world - 1) * K // world, flush=True)


if __name__ == "__main__":
    main()

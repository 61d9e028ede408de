# SPDX-License-Identifier: Apache-2.0
"""N=1 probe: where does time go when the dense sync follows / overlaps a GEMM backward?

    python scripts/overlap_probe.py [--theta BYTES]
"""
import argparse
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1902_06855_b200 import cudart  # noqa: E402
from paper_1902_06855_b200.engine import GradSync  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--theta", type=int, default=64 << 20)
    ap.add_argument("--gemms", type=int, default=80)
    args = ap.parse_args()
    torch.cuda.set_device(0)
    cudart.set_device(0)
    sizes = bench.RESNET50
    sync = GradSync(sizes, theta=args.theta)
    total = sync.layout.total
    bounds = [0]
    for s in sizes:
        bounds.append(bounds[-1] + s)
    g = [torch.randn(total, device="cuda") for _ in range(4)]
    o = [torch.empty(total, device="cuda") for _ in range(2)]

    def views(x):
        return (C.c_void_p * len(sizes))(*[x[bounds[i]:bounds[i + 1]].data_ptr() for i in range(len(sizes))])

    gp = [views(x) for x in g]
    op = [views(x) for x in o]
    A = torch.randn(2048, 4096, dtype=torch.bfloat16, device="cuda")
    B = torch.randn(4096, 4096, dtype=torch.bfloat16, device="cuda")
    Cm = torch.empty(2048, 4096, dtype=torch.bfloat16, device="cuda")
    s = torch.cuda.current_stream()
    sp = s.cuda_stream
    reps = {t: int(round(args.gemms * sizes[t - 1] / total)) for t in range(1, len(sizes) + 1)}

    def gemms(i):
        for t in range(len(sizes), 0, -1):
            for _ in range(reps[t]):
                torch.matmul(A, B, out=Cm)

    def inline(i):
        gemms(i)
        sync.dense_step(gp[i % 4], op[i % 2], stream=sp)

    def over(i):
        sync.begin_iteration(gp[i % 4], op[i % 2], stream=sp)
        for t in range(len(sizes), 0, -1):
            for _ in range(reps[t]):
                torch.matmul(A, B, out=Cm)
            sync.tensor_complete(t)
        sync.finalize_iteration()

    def sync_only(i):
        sync.dense_step(gp[i % 4], op[i % 2], stream=sp)

    def over_nogemm(i):
        sync.begin_iteration(gp[i % 4], op[i % 2], stream=sp)
        for t in range(len(sizes), 0, -1):
            sync.tensor_complete(t)
        sync.finalize_iteration()

    res = {}
    for name, fn in (("sync_only", sync_only), ("overlap_api_no_gemm", over_nogemm), ("gemms", gemms),
                     ("gemms+inline_sync", inline), ("gemms+overlap_api", over), ("gemms_again", gemms)):
        for i in range(3):
            fn(i)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        for i in range(20):
            fn(i)
        b.record(s)
        torch.cuda.synchronize()
        res[name] = round(a.elapsed_time(b) / 20, 4)
    print(json.dumps(res))


if __name__ == "__main__":
    main()

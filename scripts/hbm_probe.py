# SPDX-License-Identifier: Apache-2.0
"""HBM calibration for the N=1 dense step: what do plain torch streaming kernels reach at the
ResNet-50 gradient size, next to gf_pack / gf_unpack / the fused solo step?

    python scripts/hbm_probe.py [--elements N] [--reps R]
"""
import argparse
import ctypes as C
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_1902_06855_b200 import capi, cudart  # noqa: E402
from paper_1902_06855_b200.engine import GradSync  # noqa: E402


def timeit(fn, reps, sets):
    s = torch.cuda.current_stream()
    for i in range(3):
        fn(i % sets)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for i in range(reps):
        fn(i % sets)
    b.record(s)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3  # us


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=50)
    ap.add_argument("--workload", default="resnet50")
    args = ap.parse_args()
    torch.cuda.set_device(0)
    cudart.set_device(0)
    sizes = bench.RESNET50 if args.workload == "resnet50" else bench.ALEXNET
    sync = GradSync(sizes, theta=bench.THETA_INF)
    L = sync.layout
    n = L.total
    sets = max(2, math.ceil(2 * 126e6 / (4 * n)) + 1)
    src = [torch.randn(n, device="cuda") for _ in range(sets)]
    out = [torch.empty(n, device="cuda") for _ in range(2)]
    h16 = [torch.empty(n, device="cuda", dtype=torch.float16) for _ in range(2)]
    bounds = [0]
    for s_ in sizes:
        bounds.append(bounds[-1] + s_)

    def views(x):
        return (C.c_void_p * len(sizes))(*[x[bounds[i]:bounds[i + 1]].data_ptr() for i in range(len(sizes))])

    inp = [views(x) for x in src]
    outp = [views(x) for x in out]
    sp = torch.cuda.current_stream().cuda_stream
    res = {"elements": n, "sets": sets}
    B = n * 4

    def rec(name, us, bytes_):
        res[name] = {"us": round(us, 2), "GBps": round(bytes_ / us / 1e3, 1)}

    rec("torch_copy_f32", timeit(lambda i: out[i % 2].copy_(src[i]), args.reps, sets), 2 * B)
    rec("torch_f32_to_f16", timeit(lambda i: h16[i % 2].copy_(src[i]), args.reps, sets), 1.5 * B)
    rec("torch_f16_to_f32", timeit(lambda i: out[i % 2].copy_(h16[i % 2]), args.reps, sets), 1.5 * B)
    rec("torch_read_sum", timeit(lambda i: src[i].sum(), args.reps, sets), B)
    rec("torch_fill", timeit(lambda i: out[i % 2].fill_(1.0), args.reps, sets), B)
    m = len(sizes)

    def pack(i):
        capi.call("gf_pack", 1, sync.pool_ptr, inp[i], sync._offs, sync._cnts, m, 1.0, sp)

    def unpack(i):
        capi.call("gf_unpack", 1, sync.pool_ptr, outp[i % 2], sync._offs, sync._cnts, m, 1, sp)

    one_off = capi.u64_array([0])
    one_cnt = capi.u64_array([n])

    def pack_flat(i):
        capi.call("gf_pack", 1, sync.pool_ptr, (C.c_void_p * 1)(src[i].data_ptr()), one_off, one_cnt, 1, 1.0, sp)

    def step(i):
        pack(i)
        unpack(i)

    rec("gf_pack", timeit(pack, args.reps, sets), 1.5 * B)
    rec("gf_pack_flat", timeit(pack_flat, args.reps, sets), 1.5 * B)
    rec("gf_unpack", timeit(unpack, args.reps, sets), 1.5 * B)
    rec("gf_pack+unpack", timeit(step, args.reps, sets), 3 * B)
    rec("gf_fused_solo", timeit(lambda i: sync.fused_step(inp[i], outp[i % 2], stream=sp), args.reps, sets), 2.5 * B)
    import time
    marks = []

    def mark(name):
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        marks.append(e)

    for label, mk in (("engine_step", None), ("engine_step_marks", mark)):
        torch.cuda.synchronize()
        h0 = time.perf_counter()
        us = timeit(lambda i: sync.dense_step(inp[i], outp[i % 2], stream=sp, mark=mk), args.reps, sets)
        host = (time.perf_counter() - h0) * 1e6 / (args.reps + 3)
        rec(label, us, 3 * B)
        res[label]["host_us_incl_sync"] = round(host, 1)
    # host cost alone: enqueue while the GPU is blocked behind a long kernel
    big = torch.empty(1 << 30, device="cuda")
    for label, mk in (("enqueue_plain", None), ("enqueue_marks", mark)):
        torch.cuda.synchronize()
        big.fill_(0.0); big.fill_(1.0)
        h0 = time.perf_counter()
        for i in range(20):
            sync.dense_step(inp[i % sets], outp[i % 2], stream=sp, mark=mk)
        res[label + "_host_us_per_step"] = round((time.perf_counter() - h0) * 1e6 / 20, 1)
        torch.cuda.synchronize()
    print(json.dumps(res))


if __name__ == "__main__":
    main()

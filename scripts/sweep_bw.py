# SPDX-License-Identifier: Apache-2.0
"""fused-allreduce bandwidth sweep, 1 KB .. 1 GB of fp16, at N GPUs
(torchrun, one process per GPU). Per size, device time per call (CUDA events on the launching
stream, max over ranks) and busBW = 2(N-1)/N * bytes / t of:

  ring       gf_ring_allreduce            (push-pull, in place)
  pull       gf_ring_allreduce_unpack     (pull RS/AG + the fp32 unpack of g_avg)
  csc        gf_ring_allreduce_planned    (the CSC exchange of 10 % of the 32000-element
                                           chunks, every 10th chunk selected; busBW over the
                                           staged bytes)
  nccl       torch.distributed.all_reduce (fp16 sum, the same bytes; comparison only)

Data: zeros (every kernel here takes the same path for any finite input; values are checked
bit-exact by tests/). Prints one JSON line per size on rank 0.
    torchrun --nproc-per-node N scripts/sweep_bw.py [--max-bytes B] [--iters K]
"""
import argparse
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_1902_06855_b200 import capi, cudart  # noqa: E402
from paper_1902_06855_b200.engine import llround_pos  # noqa: E402

F16 = capi.GF_F16


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--max-bytes", type=int, default=1 << 30)
    ap.add_argument("--iters", type=int, default=20)
    args = ap.parse_args()
    rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    cudart.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    maxb = args.max_bytes
    stage_off = maxb
    heap = maxb + maxb // 8 + (1 << 20)
    comm = C.c_void_p()
    capi.call("gf_comm_create", world, rank, local, heap, C.byref(comm))
    h = (C.c_char * capi.GF_IPC_HANDLE_BYTES)()
    capi.call("gf_comm_export_handle", comm, h)
    hs = [None] * world
    dist.all_gather_object(hs, bytes(h))
    capi.call("gf_comm_connect_ipc", comm, b"".join(hs))
    base = C.c_void_p()
    capi.call("gf_comm_heap", comm, C.byref(base), None)
    cudart.memset(base.value, 0, heap)
    out = torch.empty(maxb // 2, dtype=torch.float32, device="cuda")
    nccl_buf = torch.zeros(maxb // 2, dtype=torch.float16, device="cuda")
    stream = torch.cuda.current_stream()
    sp = stream.cuda_stream

    def timed(fn, iters):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(iters):
            fn()
        e1.record(stream)
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1) / iters], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        capi.call("gf_comm_status", comm)
        return float(t.item())

    nbytes = 1 << 10
    while nbytes <= maxb:
        L = nbytes // 2
        iters = args.iters if nbytes >= (16 << 20) else 5 * args.iters
        ws, wl = capi.u64_array([0]), capi.u64_array([L])
        res = {"bytes": nbytes, "n_gpus": world}
        bus = 2 * (world - 1) / world

        t = timed(lambda: capi.call("gf_ring_allreduce", comm, F16, 0, ws, wl, 1, sp), iters)
        res["ring_us"], res["ring_busbw"] = round(t * 1e3, 2), round(bus * nbytes / (t * 1e-3) / 1e9, 1)

        dst = capi.ptr_array([out.data_ptr()])
        offs, cnts = capi.u64_array([0]), capi.u64_array([L])
        t = timed(lambda: capi.call("gf_ring_allreduce_unpack", comm, F16, 0, dst, offs, cnts, 1, ws, wl, 1,
                                    0, sp), iters)
        res["pull_unpack_us"], res["pull_unpack_busbw"] = round(t * 1e3, 2), round(bus * nbytes / (t * 1e-3) / 1e9, 1)

        chunk = 32000
        nc = max(1, llround_pos(L / chunk))
        if (nc - 1) * chunk < L:
            imp = torch.zeros(nc, dtype=torch.uint8, device="cuda")
            imp[::10] = 1
            coff = torch.zeros(nc, dtype=torch.int64, device="cuda")
            plan = torch.zeros(4 + nc, dtype=torch.int64, device="cuda")
            capi.call("gf_csc_plan", imp.data_ptr(), L, chunk, nc, F16, capi.THETA_INF, coff.data_ptr(),
                      plan.data_ptr(), sp)
            torch.cuda.synchronize()
            staged = int(plan[0].item())
            t = timed(lambda: capi.call("gf_ring_allreduce_planned", comm, F16, stage_off, plan.data_ptr(), sp),
                      iters)
            res["csc_staged_bytes"] = staged * 2
            res["csc_us"] = round(t * 1e3, 2)
            res["csc_busbw"] = round(bus * staged * 2 / (t * 1e-3) / 1e9, 1)

        x = nccl_buf[:L]
        t = timed(lambda: dist.all_reduce(x), iters)
        res["nccl_us"], res["nccl_busbw"] = round(t * 1e3, 2), round(bus * nbytes / (t * 1e-3) / 1e9, 1)
        if rank == 0:
            print(json.dumps(res), flush=True)
        nbytes *= 4
    capi.call("gf_comm_destroy", comm)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()

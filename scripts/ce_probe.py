# SPDX-License-Identifier: Apache-2.0
"""Copy-engine probe (torchrun, N GPUs): every rank PULLS a block from each peer with
cudaMemcpyAsync (peer IPC mapping -> local), all ranks at once, so every link carries traffic
in both directions — the all-gather pattern of the pull exchange. GB/s per GPU per direction
(inbound bytes / time), max time over ranks, for 1 or several streams per rank."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_1902_06855_b200 import capi, cudart  # noqa: E402

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
cudart.set_device(rank)
dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
MAXB = 256 << 20
src = torch.ones(MAXB // 2, dtype=torch.float16, device="cuda")
dst = torch.empty(world * MAXB // 2, dtype=torch.float16, device="cuda")
comm = C.c_void_p()
capi.call("gf_comm_create", world, rank, rank, 1 << 20, C.byref(comm))
h = (C.c_char * capi.GF_IPC_HANDLE_BYTES)()
capi.call("gf_comm_export_handle", comm, h)
hs = [None] * world
dist.all_gather_object(hs, bytes(h))
capi.call("gf_comm_connect_ipc", comm, b"".join(hs))
hh = (C.c_char * capi.GF_IPC_HANDLE_BYTES)()
off = C.c_uint64()
capi.call("gf_ipc_export", C.c_void_p(src.data_ptr()), hh, C.byref(off))
allh = [None] * world
dist.all_gather_object(allh, (bytes(hh), off.value))
peer = {}
for r in range(world):
    if r != rank:
        b = C.c_void_p()
        capi.call("gf_ipc_open", comm, allh[r][0], C.byref(b))
        peer[r] = b.value + allh[r][1]
streams = [torch.cuda.Stream() for _ in range(4)]
for nbytes in (8 << 20, 25 << 20, 61 << 20, 122 << 20, 256 << 20):
    for ns in (1, 2, 4):
        def go():
            k = 0
            for j in range(1, world):
                q = (rank + j) % world
                per = nbytes // ns
                for s in range(ns):
                    st = streams[k % len(streams)]
                    k += 1
                    cudart.memcpy(dst.data_ptr() + q * MAXB + s * per, peer[q] + s * per, per, st.cuda_stream)
        for _ in range(3):
            go()
        torch.cuda.synchronize()
        dist.barrier()
        cur = torch.cuda.current_stream()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(cur)
        for st in streams:
            st.wait_event(e0)
        for _ in range(10):
            go()
        for st in streams:
            ev = torch.cuda.Event()
            ev.record(st)
            cur.wait_event(ev)
        e1.record(cur)
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1) / 10], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        if rank == 0:
            gbs = (world - 1) * nbytes / (t.item() * 1e-3) / 1e9
            print(f"N={world} pull {nbytes >> 20} MiB per peer, {ns} copies per peer: "
                  f"{t.item() * 1e3:.1f} us  {gbs:.0f} GB/s inbound per GPU", flush=True)
dist.barrier()
dist.destroy_process_group()

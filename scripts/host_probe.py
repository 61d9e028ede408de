# SPDX-License-Identifier: Apache-2.0
"""Host-side cost of each C-ABI call in a dense step (diagnostic; run under torchrun)."""
import os, sys, time, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, torch.distributed as dist
from paper_1902_06855_b200 import capi, cudart
from paper_1902_06855_b200.engine import GradSync
import bench
world = int(os.environ.get("WORLD_SIZE", 1)); rank = int(os.environ.get("RANK", 0)); local = int(os.environ.get("LOCAL_RANK", 0))
torch.cuda.set_device(local); cudart.set_device(local)
if world > 1:
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
def ag(b):
    out = [None] * world; dist.all_gather_object(out, b); return out
sizes = bench.ALEXNET if (len(sys.argv) > 1 and sys.argv[1] == "alexnet") else bench.RESNET50
s = GradSync(sizes, rank=rank, world=world, device=local, allgather=ag)
tot = s.layout.total
x = torch.randn(tot, device="cuda"); y = torch.empty(tot, device="cuda")
import numpy as np
b = np.concatenate([[0], np.cumsum(sizes)])
ip = (C.c_void_p * len(sizes))(*[x[int(b[i]):int(b[i+1])].data_ptr() for i in range(len(sizes))])
op = (C.c_void_p * len(sizes))(*[y[int(b[i]):int(b[i+1])].data_ptr() for i in range(len(sizes))])
st = torch.cuda.current_stream().cuda_stream
L = s.layout
T = {"pack": 0.0, "ring": 0.0, "unpack": 0.0}
for it in range(40):
    t0 = time.perf_counter()
    capi.call("gf_pack", 1, s.pool_ptr, ip, s._offs, s._cnts, len(sizes), 1.0, st)
    t1 = time.perf_counter()
    if world > 1:
        capi.call("gf_ring_allreduce", s.comm, 1, 0, s._win[0], s._win[1], s._win[2], st)
    t2 = time.perf_counter()
    capi.call("gf_unpack", 1, s.pool_ptr, op, s._offs, s._cnts, len(sizes), world, st)
    t3 = time.perf_counter()
    if it >= 10:
        T["pack"] += t1 - t0; T["ring"] += t2 - t1; T["unpack"] += t3 - t2
torch.cuda.synchronize()
print(rank, {k: round(v / 30 * 1e6, 1) for k, v in T.items()}, "us per call", flush=True)
s.close()

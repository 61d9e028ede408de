# SPDX-License-Identifier: Apache-2.0
"""Host-side cost of each C-ABI call in a CSC step (diagnostic, 1 GPU)."""
import os, sys, time, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import numpy as np
from paper_1902_06855_b200 import capi
from paper_1902_06855_b200.engine import GradSync
import bench
torch.cuda.set_device(0)
sizes = bench.ALEXNET
s = GradSync(sizes, csc=True, theta=capi.THETA_INF, final_sparsity=0.9)
L = s.layout; nc = L.num_chunks; tot = L.total
dev = torch.device("cuda")
x = torch.randn(tot, device=dev)
b = np.concatenate([[0], np.cumsum(sizes)])
ip = (C.c_void_p * len(sizes))(*[x[int(b[i]):int(b[i+1])].data_ptr() for i in range(len(sizes))])
hg = torch.zeros(tot, device=dev); hu = torch.zeros(tot, device=dev); w = torch.zeros(tot, device=dev)
imp = [torch.ones(nc, dtype=torch.uint8, device=dev), torch.zeros(nc, dtype=torch.uint8, device=dev)]
coff = [torch.zeros(nc, dtype=torch.int64, device=dev) for _ in range(2)]
plan = [torch.zeros(4 + nc, dtype=torch.int64, device=dev) for _ in range(2)]
nacc = torch.zeros(nc, dtype=torch.int64, device=dev)
s.attach_csc_state(hg.data_ptr(), [t.data_ptr() for t in imp], [t.data_ptr() for t in coff],
                   [t.data_ptr() for t in plan], hu.data_ptr(), w.data_ptr(), nacc=nacc.data_ptr())
st = torch.cuda.current_stream().cuda_stream
s.init_csc_plan(st)
T = {}
last = [None]
def mark(name):
    t = time.perf_counter()
    if last[0] is not None:
        T[last[0][0]] = T.get(last[0][0], 0) + t - last[0][1]
    last[0] = (name, t) if name else None
for it in range(40):
    if it == 10:
        T.clear()
    s.csc_step(ip, stream=st, mark=mark)
torch.cuda.synchronize()
print({k: round(v / 30 * 1e6, 1) for k, v in T.items()}, "us per call")
t0 = time.perf_counter()
for it in range(30):
    s.csc_step(ip, stream=st)
t1 = time.perf_counter()
torch.cuda.synchronize()
print("host per step", (t1 - t0) / 30 * 1e6, "us; device-sync total", (time.perf_counter() - t0) / 30 * 1e6)

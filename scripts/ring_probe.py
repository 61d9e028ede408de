# SPDX-License-Identifier: Apache-2.0
"""In-process ring allreduce probe: N GPUs driven from one thread (gf_comm_connect_local),
busbw of gf_ring_allreduce for a sweep of sizes. Usage: python scripts/ring_probe.py N [dtype]"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1902_06855_b200 import capi  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2
dt = int(sys.argv[2]) if len(sys.argv) > 2 else 1
esz = 2 if dt == 1 else 4
heap = 512 << 20
comms = []
for r in range(n):
    c = C.c_void_p()
    capi.call("gf_comm_create", n, r, r, heap, C.byref(c))
    comms.append(c)
capi.call("gf_comm_connect_local", (C.c_void_p * n)(*[c.value for c in comms]), n)
streams = [torch.cuda.Stream(device=r) for r in range(n)]
for nbytes in [1 << 20, 4 << 20, 16 << 20, 51114064, 122201680, 256 << 20]:
    L = nbytes // esz
    ws, wl = capi.u64_array([0]), capi.u64_array([L])
    best = 1e9
    for rep in range(8):
        ev = []
        for r in range(n):
            with torch.cuda.device(r):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(streams[r])
                capi.call("gf_ring_allreduce", comms[r], dt, 0, ws, wl, 1, streams[r].cuda_stream)
                e1.record(streams[r])
                ev.append((e0, e1))
        worst = 0
        for r in range(n):
            with torch.cuda.device(r):
                ev[r][1].synchronize()
                worst = max(worst, ev[r][0].elapsed_time(ev[r][1]))
        if rep > 1:
            best = min(best, worst)
    bus = 2 * (n - 1) / n * nbytes / (best / 1e3) / 1e9
    print(f"n={n} bytes={nbytes:>11d} {best*1e3:9.1f} us  busbw {bus:7.1f} GB/s  "
          f"blocks={os.environ.get('GF_RING_BLOCKS', 'auto')}", flush=True)
for c in comms:
    capi.call("gf_comm_status", c)

# Diagnostic: colocated world on one GPU, each dense mode, trace + status.
import os, sys, time
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "..", "tests"))
import numpy as np, torch
from colo import ColoWorld, to_dev
from paper_1902_06855_b200 import capi
torch.cuda.init()
sizes = [5, 97, 1, 4099, 300_001, 8, 77, 3]
for mode in sys.argv[1:] or ["push", "pull", "rspush"]:
    for world in (2,):
        cw = ColoWorld(world, sizes, dense_mode=mode, timeout_ms=3000)
        for g in cw.ranks:
            capi.call("gf_comm_set_trace", g.comm, 1)
        gd = [to_dev(np.ones(sum(sizes), np.float32)) for _ in range(world)]
        outs = [torch.zeros(sum(sizes), device="cuda") for _ in range(world)]
        torch.cuda.synchronize()
        t0 = time.time()
        try:
            cw.dense_step(gd, outs)
            res = "ok"
        except Exception as e:
            res = repr(e)[:200]
        import ctypes as C
        tr = []
        for g in cw.ranks:
            t = (C.c_uint64 * 4)()
            capi.call("gf_comm_trace", g.comm, t)
            tr.append([t[i] - t[0] if t[i] else -1 for i in range(4)])
        print(mode, world, res, round(time.time() - t0, 2), "trace", tr, flush=True)

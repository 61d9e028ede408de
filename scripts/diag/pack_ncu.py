# Profiling harness (diagnostic): the routed pack (pack_push_kernel) of rank 0 of a colocated
# 2-rank world on ONE GPU with GF_PUSH_DIAG=2 (pack only, no barrier kernel), next to the plain
# pack (gf_pack) of the same ResNet-50 gradients. Run under ncu.
import os, sys
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")
os.environ["GF_PUSH_DIAG"] = os.environ.get("GF_PUSH_DIAG", "2")
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "..", "tests"))
import ctypes as C
import numpy as np, torch
from colo import ColoWorld, tensor_table
from paper_1902_06855_b200 import capi
from oracle.oracle import RESNET50
sizes = RESNET50
cw = ColoWorld(2, sizes, dense_mode="rspush")
g = torch.from_numpy(capi.synth_grads(0, 0, sizes)).cuda()
out = torch.empty_like(g)
gt, ot = tensor_table(g, sizes), tensor_table(out, sizes)
pool = torch.empty(sum(sizes), dtype=torch.int16, device="cuda")
offs = capi.u64_array(cw.layout.offsets)
cnts = capi.u64_array(sizes)
torch.cuda.synchronize()
for it in range(3):
    cw.ranks[0].dense_step(gt, ot)       # rank 0's routed pack only (GF_PUSH_DIAG=2)
    capi.call("gf_pack", 1, pool.data_ptr(), gt, offs, cnts, len(sizes), 1.0, None)
torch.cuda.synchronize()
print("ok")

# SPDX-License-Identifier: Apache-2.0
"""Helpers for the -m gpu tests: numpy <-> CUDA tensors (torch is only the allocator)."""
import numpy as np

try:
    import torch
except Exception:  # pragma: no cover
    torch = None

from paper_1902_06855_b200 import capi


def dev(a):
    """numpy -> CUDA tensor with identical bytes."""
    a = np.ascontiguousarray(a)
    if a.dtype == np.uint16:
        return torch.from_numpy(a.view(np.int16)).cuda()
    if a.dtype == np.uint64:
        return torch.from_numpy(a.view(np.int64)).cuda()
    return torch.from_numpy(a).cuda()


def host(t, dtype=None):
    a = t.detach().cpu().numpy()
    if dtype is not None:
        a = a.view(dtype)
    return a


def zeros(n, dtype):
    m = {np.uint16: torch.int16, np.float32: torch.float32, np.uint8: torch.uint8,
         np.uint64: torch.int64}
    return torch.zeros(int(n), dtype=m[dtype], device="cuda")


def bits(a):
    a = np.asarray(a)
    return a.view(np.uint16) if a.itemsize == 2 else a.view(np.uint32)


def sync():
    torch.cuda.synchronize()


def table(tensors):
    """(ptr array, offsets, counts) for gf_pack/gf_unpack from [(tensor, pool_off)]."""
    ptrs = capi.ptr_array([t for t, _ in tensors])
    offs = capi.u64_array([o for _, o in tensors])
    cnts = capi.u64_array([t.numel() for t, _ in tensors])
    return ptrs, offs, cnts


def pool_tensors(flat_dev, sizes, offsets):
    """Per-tensor views into a flat ascending-id fp32 device buffer + their pool offsets."""
    out, o = [], 0
    for i, s in enumerate(sizes):
        out.append((flat_dev[o:o + int(s)], int(offsets[i])))
        o += int(s)
    return out


def specials(rng, n, nan=True):
    base = rng.uniform(-1, 1, n).astype(np.float32)
    pick = rng.integers(0 if nan else 2, 12, n)
    tbl = np.array([np.nan, -np.nan, np.inf, -np.inf, 70000.0, -70000.0, 65504.0, 65520.0,
                    2.0 ** -25, 3e-8, -0.0, 1.0 + 2.0 ** -11], np.float32)
    m = rng.random(n) < 0.02
    base[m] = tbl[pick[m]]
    return base

# SPDX-License-Identifier: Apache-2.0
"""Colocated worlds: N ranks on ONE B200 running the multi-GPU kernels unchanged.

gf_comm_connect_colocated maps every rank's "peer" memory to the other ranks' allocations on
the same device, so the NVLink kernels (routed pack + rsp_kernel, pull RS/AG, push-pull ring,
CSC exchange forms, inbox selection) run with their real cross-rank flags and barriers. Each
rank launches on its own non-blocking stream; one host thread enqueues rank 0's step, then
rank 1's, ... (launches are asynchronous), then waits for all of them. A rank that never
arrives surfaces as a device-side barrier timeout (TransportError), never as a hang.
Needs CUDA_MODULE_LOADING=EAGER and CUDA_DEVICE_MAX_CONNECTIONS=32 before CUDA initialises
(tests/conftest.py sets both).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from paper_1902_06855_b200 import capi, cudart
from paper_1902_06855_b200.engine import GradSync

try:
    import torch
except Exception:  # pragma: no cover
    torch = None


def to_dev(a):
    a = np.ascontiguousarray(a)
    if a.dtype == np.uint16:
        return torch.from_numpy(a.view(np.int16)).cuda()
    return torch.from_numpy(a).cuda()


def read(ptr, nbytes, dtype, stream=None):
    out = np.empty(nbytes // np.dtype(dtype).itemsize, dtype)
    cudart.memcpy(out.ctypes.data, ptr, out.nbytes, stream)
    cudart.stream_sync(stream)
    return out


def write(ptr, arr, stream=None):
    arr = np.ascontiguousarray(arr)
    cudart.memcpy(ptr, arr.ctypes.data, arr.nbytes, stream)
    cudart.stream_sync(stream)


def tensor_table(flat, sizes):
    """ctypes pointer table of the per-tensor views of a flat ascending-id device buffer."""
    b = np.concatenate([[0], np.cumsum(np.asarray(sizes, dtype=np.int64))])
    return (C.c_void_p * len(sizes))(*[flat[int(b[i]):int(b[i + 1])].data_ptr() for i in range(len(sizes))])


class ColoWorld:
    """`world` GradSync engines on the current device, one stream per rank."""

    def __init__(self, world, sizes, **kw):
        kw.setdefault("timeout_ms", 20000)
        self.world = world
        self.sizes = [int(s) for s in sizes]
        self.ranks = GradSync.colocated(world, sizes, device=torch.cuda.current_device(), **kw)
        self.streams = [cudart.stream_create() for _ in range(world)]
        self.layout = self.ranks[0].layout

    def run(self, fn):
        """fn(rank, engine, stream) for every rank (enqueue only), then wait for all ranks."""
        for r in range(self.world):
            fn(r, self.ranks[r], self.streams[r])
        for s in self.streams:
            cudart.stream_sync(s)
        for g in self.ranks:
            g.status()

    def dense_step(self, grads, outs):
        """grads/outs: per-rank flat ascending-id device tensors."""
        gt = [tensor_table(g, self.sizes) for g in grads]
        ot = [tensor_table(o, self.sizes) for o in outs]
        self.run(lambda r, g, s: g.dense_step(gt[r], ot[r], stream=s))

    def csc_step(self, grads):
        gt = [tensor_table(g, self.sizes) for g in grads]
        self.run(lambda r, g, s: g.csc_step(gt[r], stream=s))

    def state(self, r, name, dtype):
        p, n = self.ranks[r].state(name)
        return read(p, n, dtype)

    def close(self):
        for g in self.ranks:
            g.close()
        for s in self.streams:
            cudart.stream_destroy(s)


def raw_comms(world, heap):
    """`world` bare communicators (symmetric heaps) colocated on the current device, plus one
    stream per rank and each heap's base pointer."""
    dev = torch.cuda.current_device()
    comms = []
    for r in range(world):
        c = C.c_void_p()
        capi.call("gf_comm_create", world, r, dev, heap, C.byref(c))
        capi.call("gf_comm_set_timeout_ms", c, 20000)
        comms.append(c)
    capi.call("gf_comm_connect_colocated", (C.c_void_p * world)(*[c.value for c in comms]), world)
    bases = []
    for c in comms:
        b = C.c_void_p()
        capi.call("gf_comm_heap", c, C.byref(b), None)
        bases.append(b.value)
    streams = [cudart.stream_create() for _ in range(world)]
    return comms, bases, streams


def close_raw(comms, streams):
    for s in streams:
        cudart.stream_sync(s)
        cudart.stream_destroy(s)
    for c in comms:
        capi.call("gf_comm_destroy", c)

# SPDX-License-Identifier: Apache-2.0
"""GradSync: thin Python binding of the native per-rank engine (gf_engine_*, host/engine.cpp).

The launch sequence a data-parallel trainer runs per iteration lives in C++ behind the C-ABI
(include/gflow_b200.h); this module only marshals pointers. Reference semantics (paths relative
to /root/reference/proj):

  dense (lazy allreduce, src/trainer.cpp:297-347 + src/fusion.cpp:72-109)
      world 1   one streaming pass pack -> g_avg (the collective is the identity)
      world > 1 rspush: the pack routes every vector to its segment's owner over NVLink,
                local reduce + all-gather push, unpack (pull / push-pull ring also available)
  CSC (src/sparse.cpp, Algorithm 1)
      pack+correct+compact (K2) -> exchange + write-back + exact chunk L1 (K4) ->
      norm exchange + top-k of the next set (K5) beside the momentum update (K6')

Every launch is asynchronous on the caller's stream; nothing here synchronises or reads device
memory. PoolLayout / dense_windows / sparsity_at / selection_count restate the reference's host
rules for the tests and the bench (the engine computes its own in C++).
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass

from . import capi

F32, F16 = capi.GF_F32, capi.GF_F16
THETA_INF = capi.THETA_INF
_DENSE = {"auto": capi.GF_DENSE_AUTO, "rspush": capi.GF_DENSE_RSPUSH, "pull": capi.GF_DENSE_PULL,
          "push": capi.GF_DENSE_PUSH}
_DENSE_NAME = {v: k for k, v in _DENSE.items()}
_CSC = {"push": capi.GF_CSC_PUSH, "pull": capi.GF_CSC_PULL, "auto": capi.GF_CSC_AUTO}
_CSC_NAME = {v: k for k, v in _CSC.items()}
_STATE = {"pool": capi.GF_STATE_POOL, "hg": capi.GF_STATE_HG, "hu": capi.GF_STATE_HU, "w": capi.GF_STATE_W,
          "imp_next": capi.GF_STATE_IMP_NEXT, "norms": capi.GF_STATE_NORMS, "nacc": capi.GF_STATE_NACC,
          "plan_next": capi.GF_STATE_PLAN_NEXT, "imp_cur": capi.GF_STATE_IMP_CUR, "plan_cur": capi.GF_STATE_PLAN_CUR}


def _align(x: int, a: int = 256) -> int:
    return (x + a - 1) // a * a


def llround_pos(x: float) -> int:
    """C llround for x >= 0 (half away from zero), exact for doubles < 2^52."""
    r = math.floor(x)
    return r + 1 if x - r >= 0.5 else r


@dataclass(frozen=True)
class PoolLayout:
    """GradientPool layout (src/gradient_pool.cpp:11-41): tensor m at offset 0, id 1 last;
    num_chunks = max(1, llround(total / chunk)), the last chunk absorbs the remainder."""

    sizes: tuple
    chunk: int
    offsets: tuple  # offsets[id-1]
    total: int
    num_chunks: int

    @staticmethod
    def build(sizes, chunk=32000) -> "PoolLayout":
        sizes = tuple(int(s) for s in sizes)
        if not sizes:
            raise capi.ConfigError("gradient pool needs at least one tensor")
        if chunk <= 0:
            raise capi.ConfigError("chunk_size must be positive")
        if any(s <= 0 for s in sizes):
            raise capi.ConfigError("tensor sizes must be positive")
        offs = [0] * len(sizes)
        o = 0
        for tid in range(len(sizes), 0, -1):
            offs[tid - 1] = o
            o += sizes[tid - 1]
        nc = max(1, llround_pos(o / chunk))
        return PoolLayout(sizes, chunk, tuple(offs), o, nc)

    def chunk_length(self, c: int) -> int:
        return self.total - c * self.chunk if c + 1 == self.num_chunks else self.chunk


def dense_windows(layout: PoolLayout, esz: int, theta: int):
    """FusionEngine windows of one iteration (src/fusion.cpp:72-109): tensors complete in
    descending id, a window closes when its bytes reach theta, finalize flushes the rest."""
    starts, lens = [], []
    ws = we = 0
    m = len(layout.sizes)
    for tid in range(m, -1, -1):
        flush = tid == 0
        if not flush:
            we = layout.offsets[tid - 1] + layout.sizes[tid - 1]
        hit = theta != THETA_INF and (we - ws) * esz >= theta
        if we > ws and (hit or flush):
            starts.append(ws)
            lens.append(we - ws)
            ws = we
    return starts, lens


def sparsity_at(t: int, warmup: int, final: float) -> float:
    """src/sparse.cpp:13-17"""
    if warmup == 0:
        return final
    return final * min(1.0, t / warmup)


def selection_count(sparsity: float, nc: int) -> int:
    """src/sparse.cpp:19-24 (llround, floor of one chunk)."""
    k = llround_pos((1.0 - sparsity) * nc)
    return max(1, min(k, nc))


class GradSync:
    """One rank's device-resident sync path (a gf_engine). `allgather(bytes) -> list[bytes]`
    exchanges the IPC handles when world > 1 (any control plane: torch.distributed, a TCP
    store, ...). GradSync.colocated() builds a whole world on ONE device (tests)."""

    def __init__(self, sizes, rank=0, world=1, device=0, dtype=F16, theta=64 << 20,
                 chunk=32000, csc=False, final_sparsity=0.9, warmup_iters=0, momentum=0.9,
                 lr=0.01, allgather=None, timeout_ms=30000, dense_mode="auto", csc_mode="auto",
                 _connect=True):
        if dense_mode not in _DENSE:
            raise capi.ConfigError(f"dense_mode {dense_mode!r}: auto, rspush, pull or push")
        if csc_mode not in _CSC:
            raise capi.ConfigError(f"csc_mode {csc_mode!r}: auto, pull or push")
        self.layout = PoolLayout.build(sizes, chunk)
        self.rank, self.world, self.device, self.dtype = rank, world, device, dtype
        self.esz = 2 if dtype == F16 else 4
        self.theta, self.csc = theta, csc
        self.csc_mode = csc_mode
        cfg = capi.EngineConfig()
        capi.lib().gf_engine_config_init(C.byref(cfg))
        cfg.world, cfg.rank, cfg.device, cfg.dtype = world, rank, device, dtype
        cfg.theta_bytes, cfg.chunk, cfg.csc = theta, chunk, int(bool(csc))
        cfg.dense_mode, cfg.csc_mode = _DENSE[dense_mode], _CSC[csc_mode]
        cfg.final_sparsity, cfg.warmup_iters = final_sparsity, warmup_iters
        cfg.momentum, cfg.learning_rate, cfg.timeout_ms = momentum, lr, timeout_ms
        m = len(self.layout.sizes)
        self.eng = C.c_void_p()
        capi.call("gf_engine_create", C.byref(cfg), capi.u64_array(self.layout.sizes), m, C.byref(self.eng))
        self.comm = C.c_void_p(capi.lib().gf_engine_comm(self.eng))
        if world > 1 and _connect:
            if allgather is None:
                raise capi.ConfigError("world > 1 needs an allgather for the IPC handles")
            h = (C.c_char * capi.GF_IPC_HANDLE_BYTES)()
            capi.call("gf_comm_export_handle", self.comm, h)
            capi.call("gf_engine_connect_ipc", self.eng, b"".join(allgather(bytes(h))))
        self.dense_mode = _DENSE_NAME[self.info().dense_mode] if not csc else None
        self.csc_mode = _CSC_NAME[self.info().csc_mode] if csc else None
        self._names = C.create_string_buffer(1024)
        self._ms = (C.c_float * 64)()

    @classmethod
    def colocated(cls, world, sizes, device=0, **kw):
        """`world` ranks on ONE device (gf_engine_connect_colocated): the multi-GPU kernels,
        barriers included, run unchanged; launch each rank's steps on its own stream."""
        ranks = [cls(sizes, rank=r, world=world, device=device, _connect=False, **kw) for r in range(world)]
        capi.call("gf_engine_connect_colocated", (C.c_void_p * world)(*[g.eng.value for g in ranks]), world)
        return ranks

    @classmethod
    def local(cls, world, sizes, devices=None, **kw):
        """`world` ranks in THIS process, rank r on devices[r] (peer access, gf_engine_connect_local)."""
        devices = list(range(world)) if devices is None else list(devices)
        ranks = [cls(sizes, rank=r, world=world, device=devices[r], _connect=False, **kw) for r in range(world)]
        capi.call("gf_engine_connect_local", (C.c_void_p * world)(*[g.eng.value for g in ranks]), world)
        return ranks

    def info(self):
        out = capi.EngineInfo()
        capi.call("gf_engine_info_get", self.eng, C.byref(out))
        return out

    @property
    def iteration(self):
        return int(self.info().iteration)

    def state(self, name):
        """(device pointer, bytes) of an engine buffer: pool, hg, hu, w, imp_next, imp_cur,
        norms, nacc, plan_next, plan_cur."""
        p, n = C.c_void_p(), C.c_uint64()
        capi.call("gf_engine_state", self.eng, _STATE[name], C.byref(p), C.byref(n))
        return p.value, n.value

    @property
    def pool_ptr(self):
        return self.state("pool")[0]

    last_pool_ptr = pool_ptr

    @staticmethod
    def _ptrs(ptrs):
        """Per-tensor pointer table; a prebuilt ctypes array is passed through as is."""
        if isinstance(ptrs, C.Array):
            return ptrs
        return (C.c_void_p * len(ptrs))(*ptrs)

    def dense_step(self, grad_ptrs, out_ptrs, stream=None):
        """grad_ptrs/out_ptrs: per-tensor device pointers in ascending tensor id."""
        capi.call("gf_engine_dense_step", self.eng, self._ptrs(grad_ptrs), self._ptrs(out_ptrs), stream)

    def csc_step(self, grad_ptrs, stream=None):
        """One CSC iteration (Algorithm 1) on the engine's own state buffers."""
        capi.call("gf_engine_csc_step", self.eng, self._ptrs(grad_ptrs), stream)

    # ---- overlap with backward: FusionEngine on a communication stream (fusion.cpp:25-123) ----
    def begin_iteration(self, grad_ptrs, out_ptrs, stream=None):
        capi.call("gf_engine_begin_iteration", self.eng, self._ptrs(grad_ptrs), self._ptrs(out_ptrs), stream)

    def tensor_complete(self, tid):
        capi.call("gf_engine_tensor_complete", self.eng, int(tid))

    def finalize_iteration(self):
        capi.call("gf_engine_finalize_iteration", self.eng)

    # ---- per-kernel timing ------------------------------------------------------------------
    def set_marks(self, on):
        capi.call("gf_engine_set_marks", self.eng, int(bool(on)))

    def marks(self):
        """{phase: mean ms} over the marked steps since the last call (synchronises)."""
        k = capi.lib().gf_engine_marks(self.eng, self._names, len(self._names), self._ms, len(self._ms))
        if k < 0:
            capi.check(k)
        names = self._names.value.decode().split(";") if k else []
        return {n: float(self._ms[i]) for i, n in enumerate(names)}

    def status(self):
        capi.call("gf_comm_status", self.comm)

    def close(self):
        if self.eng:
            capi.call("gf_engine_destroy", self.eng)
            self.eng = C.c_void_p()
            self.comm = C.c_void_p()

# SPDX-License-Identifier: Apache-2.0
"""ctypes binding of the C-ABI in include/gflow_b200.h.

This is exactly the binding a maintainer of a ctypes-based host would write
(see INTEGRATION.md); the pybind11 module ``gflowpy`` is the C++-API front end.
Loading fails loudly when the native library is missing — there is no
CPU fallback anywhere in the product.
"""
from __future__ import annotations

import ctypes as C
import os
import re

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
LIB_PATH = os.path.join(PKG, "libgflow_b200.so")
HEADER = os.path.join(ROOT, "include", "gflow_b200.h")

GF_OK, GF_ERR_CONFIG, GF_ERR_PROTOCOL, GF_ERR_TRANSPORT, GF_ERR_TRAINING, GF_ERR_CUDA = range(6)
GF_F32, GF_F16 = 0, 1
GF_MAX_RANKS = 16
GF_IPC_HANDLE_BYTES = 64
GF_RSAG_NO_EXIT_BARRIER = 1
GF_DENSE_AUTO, GF_DENSE_RSPUSH, GF_DENSE_PULL, GF_DENSE_PUSH = range(4)
GF_CSC_PUSH, GF_CSC_PULL, GF_CSC_AUTO = range(3)
(GF_STATE_POOL, GF_STATE_HG, GF_STATE_HU, GF_STATE_W, GF_STATE_IMP_NEXT, GF_STATE_NORMS, GF_STATE_NACC,
 GF_STATE_PLAN_NEXT, GF_STATE_IMP_CUR, GF_STATE_PLAN_CUR) = range(10)
THETA_INF = (1 << 64) - 1


class GFError(RuntimeError):
    """Base of the status-code exceptions (mirrors include/gflow/errors.hpp:11-33)."""

    status = -1


class ConfigError(GFError, ValueError):
    status = GF_ERR_CONFIG


class ProtocolError(GFError):
    status = GF_ERR_PROTOCOL


class TransportError(GFError):
    status = GF_ERR_TRANSPORT


class TrainingError(GFError):
    status = GF_ERR_TRAINING


class CudaError(TransportError):
    status = GF_ERR_CUDA


_EXC = {GF_ERR_CONFIG: ConfigError, GF_ERR_PROTOCOL: ProtocolError,
        GF_ERR_TRANSPORT: TransportError, GF_ERR_TRAINING: TrainingError, GF_ERR_CUDA: CudaError}

_vp, _u64, _i, _f = C.c_void_p, C.c_uint64, C.c_int, C.c_float
_u32 = C.c_uint32
_u64p = C.POINTER(C.c_uint64)

# name -> argtypes (restype int unless listed in _RET)
SIGNATURES = {
    "gf_encode_f16": [_vp, _vp, _u64, _f, _vp],
    "gf_decode_f16": [_vp, _vp, _u64, _vp],
    "gf_codec_digest": [_u64, _u64, _vp, _vp],
    "gf_accumulate": [_i, _vp, _vp, _u64, _vp],
    "gf_pack": [_i, _vp, _vp, _vp, _vp, _i, _f, _vp],
    "gf_unpack": [_i, _vp, _vp, _vp, _vp, _i, _i, _vp],
    "gf_chunk_norms": [_i, _vp, _u64, _u64, _u64, _vp, _i, _vp, _vp],
    "gf_csc_correct": [_i, _vp, _vp, _vp, _u64, _u64, _u64, _u64, _u64, _f, _vp],
    "gf_csc_pack_correct": [_i, _vp, _vp, _vp, _vp, _vp, _u64, _u64, _u64, _vp, _vp, _vp, _i, _f, _vp, _vp],
    "gf_csc_pack_correct_part": [_i, _vp, _vp, _vp, _vp, _vp, _vp, _u64, _u64, _u64, _vp, _vp, _vp, _i, _f, _vp,
                                 _i, _vp],
    "gf_comm_set_max_blocks": [_vp, _i],
    "gf_comm_set_block_threads": [_vp, _i],
    "gf_csc_compact": [_i, _vp, _vp, _vp, _vp, _u64, _u64, _u64, _u64, _vp],
    "gf_csc_scatter": [_i, _vp, _vp, _vp, _vp, _u64, _u64, _u64, _u64, _vp, _vp],
    "gf_csc_plan": [_vp, _u64, _u64, _u64, _i, _u64, _vp, _vp, _vp],
    "gf_select_topk": [_vp, _u64, _u64, _vp, _vp],
    "gf_csc_sgd_update": [_i, _vp, _vp, _u64, _u64, _u64, _u64, _i, _f, _f, _vp, _vp, _vp],
    "gf_dense_sgd_update": [_i, _vp, _u64, _i, _f, _f, _vp, _vp, _vp],
    "gf_comm_create": [_i, _i, _i, _u64, C.POINTER(_vp)],
    "gf_comm_destroy": [_vp],
    "gf_comm_heap": [_vp, C.POINTER(_vp), _u64p],
    "gf_comm_export_handle": [_vp, _vp],
    "gf_comm_connect_ipc": [_vp, _vp],
    "gf_comm_connect_local": [_vp, _i],
    "gf_comm_set_ring_order": [_vp, _vp],
    "gf_comm_set_timeout_ms": [_vp, _u64],
    "gf_comm_status": [_vp],
    "gf_comm_set_trace": [_vp, _i],
    "gf_comm_trace": [_vp, _vp],
    "gf_comm_trace_n": [_vp, _vp, _i],
    "gf_comm_set_select_inbox": [_vp, _u64],
    "gf_comm_set_csc_inbox": [_vp, _u64, _u64],
    "gf_csc_pack_correct_routed": [_vp, _vp, _vp, _u64, _vp, _u64, _vp, _vp, _vp, _i, _f, _vp],
    "gf_comm_rank": [_vp],
    "gf_comm_world": [_vp],
    "gf_ring_allreduce": [_vp, _i, _u64, _vp, _vp, _i, _vp],
    "gf_ring_allreduce_planned": [_vp, _i, _u64, _vp, _vp],
    "gf_ring_allreduce_planned_scatter": [_vp, _i, _u64, _vp, _vp, _u64, _u64, _vp, _vp],
    "gf_csc_exchange_pull": [_vp, _u64, _vp, _vp, _u64, _u64, _vp, _vp],
    "gf_ring_allreduce_ptrs": [_vp, _i, _vp, _vp, _vp, _i, _vp],
    "gf_sync_step_dense": [_vp, _i, _u64, _vp, _vp, _vp, _vp, _i, _vp, _vp, _i, _vp],
    "gf_sync_step_dense_push": [_vp, _i, _u64, _u64, _vp, _vp, _vp, _vp, _i, _vp, _vp, _i, _vp],
    "gf_ring_allreduce_unpack": [_vp, _i, _u64, _vp, _vp, _vp, _i, _vp, _vp, _i, _i, _vp],
    "gf_ipc_export": [_vp, _vp, _u64p],
    "gf_ipc_open": [_vp, _vp, C.POINTER(_vp)],
    "gf_ipc_close": [_vp, _vp],
    "gf_ring_allreduce_colocated": [_i, _vp, _i, _vp, _vp, _vp, _i, _vp],
    "gf_ring_allreduce_colocated_planned": [_i, _vp, _i, _vp, _vp, _vp],
    "gf_csc_select": [_vp, _u64, _u64, _u64, _vp, _u64, _u64, _i, _u64, _vp, _vp, _vp, _vp, _vp, _vp],
    "gf_csc_select_colocated": [_vp, _i, _vp, _u64, _u64, _vp, _u64, _u64, _i, _u64, _vp, _vp, _vp,
                                _vp, _vp, _vp],
    "gf_ring_traffic": [_u64, _i, _i, _i, _u64p, _u64p, _u64p],
    "gf_oracle_allreduce_ptrs": [_i, _vp, _i, _u64, _vp],
    "gf_broadcast_ptrs": [_vp, _i, _i, _u64, _vp],
    "gf_ring_reduce_ptrs": [_i, _vp, _i, _i, _u64, _vp],
    "gf_comm_connect_colocated": [_vp, _i],
    "gf_synth_grads": [_i, _i, _vp, _i, _vp],
    "gf_engine_config_init": [_vp],
    "gf_engine_create": [_vp, _vp, _i, C.POINTER(_vp)],
    "gf_engine_destroy": [_vp],
    "gf_engine_comm": [_vp],
    "gf_engine_connect_ipc": [_vp, _vp],
    "gf_engine_connect_local": [_vp, _i],
    "gf_engine_connect_colocated": [_vp, _i],
    "gf_engine_info_get": [_vp, _vp],
    "gf_engine_state": [_vp, _i, C.POINTER(_vp), _u64p],
    "gf_engine_dense_step": [_vp, _vp, _vp, _vp],
    "gf_engine_csc_step": [_vp, _vp, _vp],
    "gf_engine_begin_iteration": [_vp, _vp, _vp, _vp],
    "gf_engine_tensor_complete": [_vp, _i],
    "gf_engine_finalize_iteration": [_vp],
    "gf_engine_set_marks": [_vp, _i],
    "gf_engine_marks": [_vp, _vp, _i, _vp, _i],
    "gf_abi_version": [],
    "gf_last_error": [],
    "gf_kernel_launches": [],
}
_RET = {"gf_last_error": C.c_char_p, "gf_kernel_launches": C.c_uint64, "gf_engine_config_init": None,
        "gf_engine_comm": C.c_void_p}


class EngineConfig(C.Structure):
    """gf_engine_config (include/gflow_b200.h)."""
    _fields_ = [("world", C.c_int), ("rank", C.c_int), ("device", C.c_int), ("dtype", C.c_int),
                ("theta_bytes", C.c_uint64), ("chunk", C.c_uint64), ("csc", C.c_int),
                ("dense_mode", C.c_int), ("csc_mode", C.c_int), ("final_sparsity", C.c_double),
                ("warmup_iters", C.c_uint64), ("momentum", C.c_double), ("learning_rate", C.c_double),
                ("timeout_ms", C.c_uint64)]


class EngineInfo(C.Structure):
    """gf_engine_info (include/gflow_b200.h)."""
    _fields_ = [("total", C.c_uint64), ("num_chunks", C.c_uint64), ("heap_bytes", C.c_uint64),
                ("nwin", C.c_int), ("dense_mode", C.c_int), ("iteration", C.c_uint64), ("csc_mode", C.c_int)]


def header_symbols() -> list[str]:
    """Every function the public header declares."""
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"^(?:int|const char\*|uint64_t|void|gf_comm\*)\s+(gf_[a-z0-9_]+)\s*\(", txt,
                                 re.M)))


_lib = None


def lib():
    """Load the native library (raises if it was not built — no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_1902_06855_b200.build`")
        L = C.CDLL(LIB_PATH)
        for name, args in SIGNATURES.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = _RET.get(name, C.c_int)
        _lib = L
    return _lib


def check(rc: int) -> None:
    if rc != GF_OK:
        msg = lib().gf_last_error().decode(errors="replace")
        raise _EXC.get(rc, GFError)(f"[gf status {rc}] {msg}")


def call(name: str, *args) -> None:
    check(getattr(lib(), name)(*args))


def ptr(t) -> int:
    """Device/host pointer of a torch tensor, numpy array, int or None."""
    if t is None:
        return None
    if isinstance(t, int):
        return t
    if hasattr(t, "data_ptr"):
        return t.data_ptr()
    if hasattr(t, "ctypes"):
        return t.ctypes.data
    raise TypeError(type(t))


def u64_array(vals):
    arr = (C.c_uint64 * len(vals))(*[int(v) for v in vals])
    return arr


def synth_grads(rank, step, sizes):
    """SURVEY §8(d) seeded gradients (gf_synth_grads) as a flat ascending-id float32 array."""
    import numpy as np
    out = np.empty(int(sum(int(s) for s in sizes)), dtype=np.float32)
    call("gf_synth_grads", int(rank), int(step), u64_array(sizes), len(sizes), out.ctypes.data)
    return out


def ptr_array(ptrs):
    return (C.c_void_p * len(ptrs))(*[ptr(p) for p in ptrs])


def int_array(vals):
    return (C.c_int * len(vals))(*[int(v) for v in vals])

# SPDX-License-Identifier: Apache-2.0
"""Minimal ctypes access to the CUDA runtime the native library links against.

Used by the engine/bench/tests to move bytes in and out of the symmetric heap
(which gf_comm_create allocates with cudaMalloc, outside PyTorch's allocator).
Only plain cudaMemcpyAsync / cudaMemsetAsync / stream & event calls.
"""
from __future__ import annotations

import ctypes as C
import os

# soname first: resolves to the runtime instance torch / libgflow_b200 already loaded
_CANDIDATES = ["libcudart.so.12", "/usr/local/cuda/lib64/libcudart.so.12", "libcudart.so"]
cudaMemcpyDefault = 4
_rt = None


def rt():
    global _rt
    if _rt is None:
        last = None
        for p in _CANDIDATES:
            try:
                _rt = C.CDLL(p)
                break
            except OSError as e:  # pragma: no cover
                last = e
        if _rt is None:
            raise ImportError(f"libcudart not found: {last}")
        _rt.cudaMemcpyAsync.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_int, C.c_void_p]
        _rt.cudaMemsetAsync.argtypes = [C.c_void_p, C.c_int, C.c_size_t, C.c_void_p]
        _rt.cudaStreamSynchronize.argtypes = [C.c_void_p]
        _rt.cudaGetErrorString.restype = C.c_char_p
        _rt.cudaSetDevice.argtypes = [C.c_int]
        _rt.cudaHostRegister.argtypes = [C.c_void_p, C.c_size_t, C.c_uint]
        _rt.cudaHostUnregister.argtypes = [C.c_void_p]
        _rt.cudaStreamCreateWithFlags.argtypes = [C.POINTER(C.c_void_p), C.c_uint]
        _rt.cudaEventCreateWithFlags.argtypes = [C.POINTER(C.c_void_p), C.c_uint]
        _rt.cudaEventRecord.argtypes = [C.c_void_p, C.c_void_p]
        _rt.cudaStreamWaitEvent.argtypes = [C.c_void_p, C.c_void_p, C.c_uint]
        _rt.cudaStreamDestroy.argtypes = [C.c_void_p]
    return _rt


def _chk(rc, what):
    if rc != 0:
        raise RuntimeError(f"{what}: {rt().cudaGetErrorString(rc).decode()}")


def memcpy(dst: int, src: int, nbytes: int, stream: int | None = None) -> None:
    _chk(rt().cudaMemcpyAsync(C.c_void_p(dst), C.c_void_p(src), nbytes, cudaMemcpyDefault,
                              C.c_void_p(stream or 0)), "cudaMemcpyAsync")


def memset(dst: int, value: int, nbytes: int, stream: int | None = None) -> None:
    _chk(rt().cudaMemsetAsync(C.c_void_p(dst), value, nbytes, C.c_void_p(stream or 0)),
         "cudaMemsetAsync")


def stream_create() -> int:
    """A non-blocking stream on the current device (never destroyed: engine lifetime)."""
    h = C.c_void_p()
    _chk(rt().cudaStreamCreateWithFlags(C.byref(h), 1), "cudaStreamCreateWithFlags")
    return h.value


def stream_destroy(s: int) -> None:
    _chk(rt().cudaStreamDestroy(C.c_void_p(s)), "cudaStreamDestroy")


def stream_sync(s: int | None) -> None:
    _chk(rt().cudaStreamSynchronize(C.c_void_p(s or 0)), "cudaStreamSynchronize")


def event_create() -> int:
    h = C.c_void_p()
    _chk(rt().cudaEventCreateWithFlags(C.byref(h), 2), "cudaEventCreateWithFlags")  # no timing
    return h.value


def event_record(ev: int, stream: int | None) -> None:
    _chk(rt().cudaEventRecord(C.c_void_p(ev), C.c_void_p(stream or 0)), "cudaEventRecord")


def stream_wait(stream: int | None, ev: int) -> None:
    _chk(rt().cudaStreamWaitEvent(C.c_void_p(stream or 0), C.c_void_p(ev), 0), "cudaStreamWaitEvent")


def sync_device() -> None:
    _chk(rt().cudaDeviceSynchronize(), "cudaDeviceSynchronize")


def set_device(d: int) -> None:
    _chk(rt().cudaSetDevice(d), "cudaSetDevice")


_ = os  # keep import for future env overrides

# SPDX-License-Identifier: Apache-2.0
"""B200-native gradient-synchronisation path of GradientFlow (arXiv 1902.06855).

Layers:
  include/gflow_b200.h            C-ABI drop-in boundary (plain pointers, status codes)
  csrc/*.cu                       sm_100a kernels: pack, CSC (correct/norm/select/compact),
                                  NVLink peer-memory ring allreduce, unpack
  csrc/include/gflow/*.hpp        the reference's C++ API (GradientPool, FusionEngine,
                                  SparseState, ring_allreduce, ...) re-implemented on the GPU
  gflowpy (pybind11)              the reference's Python bindings, same names/kwargs
  capi.py / engine.py             ctypes binding and the multi-process GradSync engine
"""
from . import capi  # noqa: F401

__all__ = ["capi"]

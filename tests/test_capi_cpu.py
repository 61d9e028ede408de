# SPDX-License-Identifier: Apache-2.0
"""CPU: the C-ABI library loads and exports every symbol include/gflow_b200.h declares.

No kernel is launched here (no GPU in the build container); only host-side
arithmetic entry points and argument validation that fails before any CUDA call.
"""
import ctypes as C

import pytest

from paper_1902_06855_b200 import capi


def test_library_exports_every_header_symbol():
    L = capi.lib()
    declared = capi.header_symbols()
    assert len(declared) >= 30
    missing = [s for s in declared if not hasattr(L, s)]
    assert not missing, missing
    # the ctypes table covers the whole header too
    assert sorted(capi.SIGNATURES) == declared


def test_abi_version():
    assert capi.lib().gf_abi_version() == 1


def test_ring_traffic_law_host_only():
    # test_collectives.cpp:73-100: per-rank payload 2(N-1)K/N; N=4, K=1 KiB -> 1536 B
    for n in (1, 2, 3, 4, 8):
        for elems in (1, 97, 1024, 1 << 18):
            tot = 0
            for pos in range(n):
                s, r, f = C.c_uint64(), C.c_uint64(), C.c_uint64()
                capi.call("gf_ring_traffic", elems, n, pos, capi.GF_F16, C.byref(s), C.byref(r),
                          C.byref(f))
                assert f.value == 2 * (n - 1)
                tot += s.value
                if elems % n == 0:
                    assert s.value == 2 * (n - 1) * elems * 2 // n
            # every element leaves its owner (n-1) times in RS and in AG
            assert tot == (2 * (n - 1) * elems * 2 if n > 1 else 0)


def test_config_errors_map_to_exceptions():
    with pytest.raises(capi.ConfigError):
        capi.call("gf_pack", 9, None, None, None, None, 0, 1.0, None)
    with pytest.raises(capi.ConfigError):
        capi.call("gf_ring_traffic", 10, 0, 0, 1, None, None, None)
    with pytest.raises(ValueError):  # ConfigError is-a ValueError, like gflowpy
        capi.call("gf_ring_allreduce_colocated", 1, None, 0, None, None, None, 0, None)
    with pytest.raises(capi.ConfigError):
        capi.call("gf_comm_create", 4, 7, 0, 1024, C.byref(C.c_void_p()))


def test_engine_config_defaults():
    """gf_engine_config_init: the reference's defaults (fusion.hpp:27-30 theta 64 MiB,
    gradient_pool.hpp:16 chunk 32000, sparse.hpp:21-26 momentum 0.9 / lr 0.01, transport.hpp:25
    timeout 30 s); host-only."""
    cfg = capi.EngineConfig()
    capi.lib().gf_engine_config_init(C.byref(cfg))
    assert (cfg.world, cfg.rank, cfg.dtype, cfg.theta_bytes, cfg.chunk) == (1, 0, capi.GF_F16, 64 << 20, 32000)
    assert (cfg.csc, cfg.dense_mode, cfg.csc_mode) == (0, capi.GF_DENSE_AUTO, capi.GF_CSC_AUTO)
    assert (cfg.momentum, cfg.learning_rate, cfg.timeout_ms) == (0.9, 0.01, 30000)
    with pytest.raises(capi.ConfigError):
        capi.call("gf_engine_create", C.byref(cfg), capi.u64_array([]), 0, C.byref(C.c_void_p()))
    cfg.chunk = 0
    with pytest.raises(capi.ConfigError):
        capi.call("gf_engine_create", C.byref(cfg), capi.u64_array([5]), 1, C.byref(C.c_void_p()))


def test_synth_grads_match_reference_stream(reference):
    """gf_synth_grads (host) is the reference's seeded generator (the stream
    oracle/ref_driver.cpp draws with the reference build): bit-identical values, so bench.py's
    GPU arm and its CPU reference arm sync the same gradients."""
    import numpy as np
    sizes = [23232, 64, 307200, 192, 7, 1000]
    for r, t in ((0, 0), (3, 1), (7, 5)):
        a = capi.synth_grads(r, t, sizes)
        b = reference.gen_grads(r, t, sizes)
        assert (a.view(np.uint32) == b.view(np.uint32)).all(), (r, t)

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

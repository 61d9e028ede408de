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


def test_part_ranges_tile_every_segment():
    """gf_part_ranges (host-only): the pieces of a pull-mode step are disjoint, tile every
    window exactly, and cut segments at multiples of 8 elements (16-byte fp16 vectors)."""
    import numpy as np
    rng = np.random.default_rng(3)
    for world in (2, 3, 4, 8):
        for _ in range(20):
            nwin = int(rng.integers(1, 6))
            wl = rng.integers(1, 200_000, nwin).tolist()
            ws = np.concatenate([[0], np.cumsum(wl)[:-1]]).tolist()
            cuts = sorted(set([0, 1024] + rng.integers(1, 1024, int(rng.integers(0, 4))).tolist()))
            cover = np.zeros(sum(wl), np.int32)
            for lo_q, hi_q in zip(cuts, cuts[1:]):
                lo, hi = capi.part_ranges(ws, wl, world, lo_q, hi_q)
                assert (lo < hi).all() and (lo[1:] >= hi[:-1]).all()
                for a, b in zip(lo.tolist(), hi.tolist()):
                    cover[a:b] += 1
                    # a cut point inside a segment is 8-aligned
                    seg_edges = set()
                    for s0, l in zip(ws, wl):
                        base, rem = divmod(l, world)
                        for j in range(world + 1):
                            seg_edges.add(s0 + j * base + min(j, rem))
                    assert a in seg_edges or a % 8 == 0
                    assert b in seg_edges or b % 8 == 0
            assert (cover == 1).all()
    with pytest.raises(capi.ConfigError):
        capi.part_ranges([0], [10], 2, 5, 4)

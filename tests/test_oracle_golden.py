# SPDX-License-Identifier: Apache-2.0
"""CPU: pin the C restatement (oracle/gf_oracle.c) to the reference.

Golden fixtures in tests/golden/ were produced by the UNMODIFIED reference library
(tests/golden/gen_golden.py); the KATs below restate the reference's own unit tests
(file:line cited). When oracle/_ref is present the restatement is also compared
against the live reference on fresh random inputs.
"""
import numpy as np
import pytest

from oracle.oracle import ALEXNET, RESNET50, THETA_INF


def bits(a):
    a = np.asarray(a)
    return a.view(np.uint16) if a.dtype == np.uint16 else a.view(np.uint32)


# ---- codec: test_half.cpp:15-107 -------------------------------------------------
def test_codec_kats(oracle, golden):
    g = golden("codec_layout.npz")
    assert (oracle.f2h(g["kat_in"]) == g["kat_out"]).all()
    assert oracle.f2h([0.0])[0] == 0x0000 and oracle.f2h([-0.0])[0] == 0x8000  # :15-20
    assert oracle.f2h([1.0])[0] == 0x3C00                                      # :22-25
    assert list(oracle.f2h([70000.0, -70000.0, np.inf])) == [0x7BFF, 0xFBFF, 0x7BFF]  # :27-38
    assert oracle.f2h([np.nan])[0] & 0x7E00 == 0x7E00
    assert oracle.f2h([1 + 2.0 ** -11])[0] == 0x3C00                           # :72-80 ties-to-even
    assert oracle.f2h([1 + 3 * 2.0 ** -11])[0] == 0x3C02
    assert oracle.h2f([0x0001])[0] == 2.0 ** -24                               # :101-107


def test_decode_exhaustive(oracle, golden):
    g = golden("codec_layout.npz")
    h = np.arange(65536, dtype=np.uint16)
    assert (bits(oracle.h2f(h)) == g["decode_table_bits"]).all()


def test_encode_round_trip_all_finite_halves(oracle):
    # test_half.cpp:40-56: every finite half survives decode->encode
    h = np.arange(65536, dtype=np.uint16)
    finite = (h & 0x7C00) != 0x7C00
    assert (oracle.f2h(oracle.h2f(h[finite])) == h[finite]).all()


def test_encode_digest_slice_matches_reference(oracle, golden):
    # Two of the 64 reference slices of the exhaustive 2^32 digest (the full sweep runs
    # on the GPU, tests/test_gpu_codec.py, where the device encoder is checked).
    g = golden("codec_layout.npz")
    per = (1 << 32) // 64
    for i in (0, 47):  # +0..small, and a slice inside the negative range
        assert oracle.codec_digest(i * per, per, nthreads=4) == int(g["codec_digest_slices"][i])


def test_accumulate(oracle, golden):
    g = golden("codec_layout.npz")
    d, src = g["acc_a"].copy(), g["acc_b"]  # keep src alive while C reads it
    oracle.L.go_accumulate(1, d.ctypes.data, src.ctypes.data, d.size)
    assert (d == g["acc_out"]).all()
    d32, src32 = g["acc32_a"].copy(), g["acc32_b"]
    oracle.L.go_accumulate(0, d32.ctypes.data, src32.ctypes.data, d32.size)
    assert (bits(d32) == bits(g["acc32_out"])).all()


# ---- layout: test_pool.cpp:15-66 ------------------------------------------------------
def test_pool_layout_kats(oracle, golden):
    assert oracle.pool_layout([60900000], 32000)[1] == 1903
    assert oracle.pool_layout([25500000], 32000)[1] == 797
    off, nc, lens = oracle.pool_layout([3, 2, 1], 4)
    assert list(off) == [3, 1, 0]
    off, nc, lens = oracle.pool_layout([10], 4)
    assert nc == 3 and list(lens) == [4, 4, 2]
    assert list(oracle.pool_layout([70000], 32000)[2]) == [32000, 38000]
    assert oracle.pool_layout([3], 100)[1] == 1
    g = golden("codec_layout.npz")
    for name, sizes in (("alexnet", ALEXNET), ("resnet50", RESNET50)):
        off, nc, lens = oracle.pool_layout(sizes, 32000)
        assert (off == g[f"{name}_offsets"]).all()
        assert nc == int(g[f"{name}_nc"][0])
        assert (lens == g[f"{name}_chunk_lens"]).all()
    assert oracle.pool_layout(ALEXNET, 32000)[1] == 1909
    assert oracle.pool_layout(RESNET50, 32000)[1] == 799


def test_selection_count_kats(oracle, golden):
    g = golden("codec_layout.npz")
    for s, nc, k in zip(g["selcount_s"], g["selcount_nc"], g["selcount_k"]):
        assert oracle.selection_count(float(s), int(nc)) == int(k)
    assert oracle.selection_count(0.85, 1903) == 285  # test_sparse.cpp:76
    assert oracle.selection_count(0.9, 1903) == 190
    assert oracle.sparsity_at(5, 10, 0.9) == pytest.approx(0.45)
    assert oracle.sparsity_at(25, 10, 0.85) == 0.85


def test_selection_hand_traces(oracle, golden):
    g = golden("codec_layout.npz")
    # test_sparse.cpp:198-216: summed norms [2,0,2,4], k=2 -> {0,3}
    assert list(oracle.select_topk(np.array([2, 0, 2, 4], np.float32), 2)) == list(g["trace_bitset"])
    # :218-233 ties -> lowest indices
    assert list(oracle.select_topk(np.array([3, 3, 3, 3], np.float32), 2)) == list(g["trace_ties"])


# ---- dense lazy allreduce: fusion.cpp + collectives.cpp ---------------------------------
def test_dense_sync_golden(oracle, golden):
    g = golden("dense_sync.npz")
    for ci in range(int(g["dense_cases"][0])):
        p = f"d{ci}_"
        n, dt, theta = (int(x) for x in g[p + "meta"])
        sizes = g[p + "sizes"]
        esz = 2 if dt == 1 else 4
        ws, wl = oracle.dense_windows(sizes, esz, theta)
        assert list(wl * esz) == list(g[p + "window_bytes"]), ci
        pools = [oracle.pack(gr, sizes, dtype=dt) for gr in g[p + "grads"]]
        oracle.ring_allreduce(pools, dtype=dt, windows=(ws, wl))
        for r in range(n):
            assert (bits(pools[r]) == bits(g[p + "pools"][r])).all(), (ci, r)
            assert (bits(oracle.unpack(pools[r], n, dtype=dt)) == bits(g[p + "gavg"][r])).all()


# ---- CSC: sparse.cpp ------------------------------------------------------------------
def test_csc_golden(oracle, golden):
    g = golden("csc_run.npz")
    for ci in range(int(g["csc_cases"][0])):
        p = f"c{ci}_"
        n, dt, theta, chunk, T = (int(x) for x in g[p + "meta"])
        sizes = g[p + "sizes"]
        total = int(sizes.sum())
        nc = oracle.pool_layout(sizes, chunk)[1]
        hg = [np.zeros(total, np.float32) for _ in range(n)]
        imp = np.ones(nc, np.uint8)
        for t in range(T):
            assert (g[p + "imp"][t][0] == imp).all()
            assert oracle.fnv1a(imp) == int(g[p + "checksum"][t][0])
            k = oracle.selection_count(oracle.sparsity_at(t + 1, 2, 0.75), nc)
            pools, norms, nxt, nw = oracle.csc_iteration(list(g[p + "grads"][t]), sizes, chunk,
                                                         theta, np.float32(0.9), imp, k, hg, dtype=dt)
            assert nw == int(g[p + "windows"][t][0])
            for r in range(n):
                assert (bits(hg[r]) == bits(g[p + "hg"][t][r])).all(), (ci, t, r)
                assert (bits(pools[r]) == bits(g[p + "pool_x"][t][r])).all(), (ci, t, r)
                assert (bits(norms[r]) == bits(g[p + "norms_sum"][t][r])).all(), (ci, t, r)
                assert (nxt == g[p + "next_imp"][t][r]).all()
            imp = nxt


def test_csc_sgd_update_golden(oracle, golden):
    g = golden("csc_run.npz")
    p = "c0_"
    n, dt, theta, chunk, T = (int(x) for x in g[p + "meta"])
    total = int(g[p + "sizes"].sum())
    for r in range(n):
        hu = np.zeros(total, np.float32)
        w = g[p + "w0"].copy()
        for t in range(T):
            oracle.csc_sgd_update(g[p + "pool_x"][t][r], g[p + "imp"][t][r], chunk, n,
                                  np.float32(0.9), np.float32(0.01), hu, w, dtype=dt)
            assert (bits(hu) == bits(g[p + "hu"][t][r])).all()
            assert (bits(w) == bits(g[p + "w"][t][r])).all()


# ---- live reference cross-check (fresh random inputs) ----------------------------------
def test_restatement_vs_live_reference(oracle, reference):
    rng = np.random.default_rng(1234)
    x = rng.integers(0, 2 ** 32, 1 << 20, dtype=np.uint64).astype(np.uint32).view(np.float32)
    assert (oracle.f2h(x) == reference.f2h(x)).all()
    for n in (2, 3, 5, 8):
        for L in (1, 7, 97, 4099):
            for dt in (0, 1):
                v = [rng.uniform(-1, 1, L).astype(np.float32) * 100 for _ in range(n)]
                a = [oracle.f2h(z) if dt else z.copy() for z in v]
                b = [z.copy() for z in a]
                ring = rng.permutation(n).astype(np.int32)
                oracle.ring_allreduce(a, dtype=dt, ring_order=ring)
                reference.allreduce(b, dtype=dt, ring_order=ring)
                for r in range(n):
                    assert (bits(a[r]) == bits(b[r])).all()


def test_windows_vs_live_reference(oracle, reference):
    rng = np.random.default_rng(99)
    for _ in range(20):
        sizes = list(rng.integers(1, 5000, rng.integers(1, 12)))
        theta = int(rng.choice([0, 64, 1000, 8192, THETA_INF]))
        grads = [rng.uniform(-1, 1, sum(sizes)).astype(np.float32)]
        _, _, wb, _ = reference.dense_sync(grads, sizes, dtype=1, theta=theta)
        _, wl = oracle.dense_windows(sizes, 2, theta)
        assert list(wl * 2) == list(wb)


def test_nan_propagation_vs_live_reference(oracle, reference):
    """Both-NaN accumulations keep the operand the reference's binary keeps (fp16: incoming,
    fp32: local) — pinned on NaN-dense data with both signs."""
    rng = np.random.default_rng(0)

    def nan_dense(n):
        x = rng.uniform(-1, 1, n).astype(np.float32)
        m = rng.random(n) < 0.3
        b = x.view(np.uint32).copy()
        b[m] = 0x7FC00000 | (rng.integers(0, 2, int(m.sum())).astype(np.uint32) << 31)
        return b.view(np.float32)
    for n in (2, 3, 4, 8):
        for dt in (0, 1):
            v = [nan_dense(5000) for _ in range(n)]
            a = [oracle.f2h(z) if dt else z.copy() for z in v]
            b = [z.copy() for z in a]
            oracle.ring_allreduce(a, dtype=dt)
            reference.allreduce(b, dtype=dt)
            for r in range(n):
                assert (bits(a[r]) == bits(b[r])).all()


# ---- rooted collectives: reduce() and hierarchical_allreduce() ---------------------------
def test_rooted_golden(oracle, golden):
    """Oracle restatement vs the reference's reduce() end state on EVERY rank (the root's
    sums and the reduce-scatter partials elsewhere) and its hierarchical_allreduce."""
    import json
    g = golden("rooted.npz")
    cases = json.loads(str(g["cases_json"]))
    for i, (n, dt, length, root, ring) in enumerate(cases["reduce"]):
        bufs = [x.copy() for x in g[f"r{i}_in"]]
        oracle.ring_reduce(bufs, root, dtype=dt, ring_order=ring)
        for r in range(n):
            assert (bits(bufs[r]) == bits(g[f"r{i}_out"][r])).all(), (i, r)
    for i, (n, m, dt, length) in enumerate(cases["hier"]):
        bufs = [x.copy() for x in g[f"h{i}_in"]]
        oracle.hier_allreduce(bufs, m, dtype=dt)
        for r in range(n):
            assert (bits(bufs[r]) == bits(g[f"h{i}_out"][r])).all(), (i, r)

# SPDX-License-Identifier: Apache-2.0
"""GPU parity: every sm_100a kernel vs the oracle / reference golden vectors, bit-exact.

All calls go through the C-ABI (include/gflow_b200.h) via ctypes.
"""
import ctypes as C

import numpy as np
import pytest

from oracle.oracle import ALEXNET, RESNET50, THETA_INF

pytestmark = pytest.mark.gpu

F16, F32 = 1, 0


@pytest.fixture(scope="module")
def G():
    import gpu_util as G
    return G


# ---- codec ---------------------------------------------------------------------------
def test_codec_exhaustive_digest(gf, golden, G):
    """Device encoder over all 2^32 fp32 patterns == reference float_to_half_bits."""
    g = golden("codec_layout.npz")
    d = G.zeros(1, np.uint64)
    gf.call("gf_codec_digest", 0, 1 << 32, d.data_ptr(), None)
    G.sync()
    assert int(G.host(d, np.uint64)[0]) == int(g["codec_digest_all"][0])
    # slices too (localises a failure)
    per = (1 << 32) // 64
    for i in (0, 31, 32, 63):
        d.zero_()
        gf.call("gf_codec_digest", i * per, per, d.data_ptr(), None)
        G.sync()
        assert int(G.host(d, np.uint64)[0]) == int(g["codec_digest_slices"][i]), i


def test_decode_exhaustive(gf, golden, G):
    g = golden("codec_layout.npz")
    h = G.dev(np.arange(65536, dtype=np.uint16))
    out = G.zeros(65536, np.float32)
    gf.call("gf_decode_f16", h.data_ptr(), out.data_ptr(), 65536, None)
    G.sync()
    assert (G.bits(G.host(out)) == g["decode_table_bits"]).all()


def test_encode_kats_and_specials(gf, golden, oracle, G):
    g = golden("codec_layout.npz")
    rng = np.random.default_rng(3)
    for x in (g["kat_in"], G.specials(rng, 1 << 20) * 3e4):
        xd = G.dev(x.astype(np.float32))
        out = G.zeros(x.size, np.uint16)
        gf.call("gf_encode_f16", xd.data_ptr(), out.data_ptr(), x.size, 1.0, None)
        G.sync()
        assert (G.host(out, np.uint16) == oracle.f2h(x)).all()


def test_accumulate(gf, golden, G):
    g = golden("codec_layout.npz")
    d = G.dev(g["acc_a"])
    src = G.dev(g["acc_b"])  # keep device temporaries alive across the async call
    gf.call("gf_accumulate", F16, d.data_ptr(), src.data_ptr(), d.numel(), None)
    G.sync()
    assert (G.host(d, np.uint16) == g["acc_out"]).all()
    d32 = G.dev(g["acc32_a"])
    s32 = G.dev(g["acc32_b"])
    gf.call("gf_accumulate", F32, d32.data_ptr(), s32.data_ptr(), d32.numel(), None)
    G.sync()
    assert (G.bits(G.host(d32)) == G.bits(g["acc32_out"])).all()


# ---- K1 pack / K6 unpack ----------------------------------------------------------------
@pytest.mark.parametrize("name,sizes", [("alexnet", ALEXNET), ("resnet50", RESNET50),
                                        ("ragged", [13, 29, 7, 41, 11, 8191, 1, 3])])
@pytest.mark.parametrize("dtype", [F16, F32])
def test_pack_unpack_parity(gf, oracle, G, name, sizes, dtype):
    off, nc, _ = oracle.pool_layout(sizes, 32000)
    rng = np.random.default_rng(len(sizes) + dtype)
    flat = oracle.gen_grads(7, sizes) * np.float32(3.0)
    flat[rng.integers(0, flat.size, 64)] = np.float32(np.inf)
    flat[rng.integers(0, flat.size, 64)] = np.float32(-7e4)
    flat[rng.integers(0, flat.size, 64)] = np.float32(np.nan)
    flat[rng.integers(0, flat.size, 64)] = np.float32(3e-8)
    fd = G.dev(flat)
    total = int(sum(sizes))
    pool = G.zeros(total, np.uint16 if dtype == F16 else np.float32)
    ptrs, offs, cnts = G.table(G.pool_tensors(fd, sizes, off))
    gf.call("gf_pack", dtype, pool.data_ptr(), ptrs, offs, cnts, len(sizes), 1.0, None)
    G.sync()
    want = oracle.pack(flat, sizes, dtype=dtype)
    got = G.host(pool, np.uint16 if dtype == F16 else np.float32)
    assert (G.bits(got) == G.bits(want)).all()
    # unpack with 1/N, N = 3 (inexact reciprocal) and 4
    for world in (3, 4):
        outs = G.zeros(total, np.float32)
        uptrs, uoffs, ucnts = G.table(G.pool_tensors(outs, sizes, off))
        gf.call("gf_unpack", dtype, pool.data_ptr(), uptrs, uoffs, ucnts, len(sizes), world, None)
        G.sync()
        want_g = oracle.unpack(want, world, dtype=dtype)  # pool order
        got_pool_order = np.empty(total, np.float32)
        o = 0
        h = G.host(outs)
        for i, s in enumerate(sizes):
            got_pool_order[int(off[i]):int(off[i]) + s] = h[o:o + s]
            o += s
        assert (G.bits(got_pool_order) == G.bits(want_g)).all(), world


def test_pack_misaligned_sources(gf, oracle, G):
    """Tensor base pointers off 16-B alignment and odd pool offsets take the scalar path."""
    sizes = [5, 1031, 17, 4099, 2]
    off, _, _ = oracle.pool_layout(sizes, 1000)
    flat = oracle.gen_grads(3, sizes)
    big = G.dev(np.concatenate([np.zeros(1, np.float32), flat]))  # shift by 4 bytes
    fd = big[1:]
    pool = G.zeros(sum(sizes), np.uint16)
    ptrs, offs, cnts = G.table(G.pool_tensors(fd, sizes, off))
    gf.call("gf_pack", F16, pool.data_ptr(), ptrs, offs, cnts, len(sizes), 1.0, None)
    G.sync()
    assert (G.host(pool, np.uint16) == oracle.pack(flat, sizes, dtype=F16)).all()


def test_pack_scale_power_of_two(gf, oracle, G):
    sizes = [4096, 100]
    off, _, _ = oracle.pool_layout(sizes, 1000)
    flat = oracle.gen_grads(4, sizes)
    fd = G.dev(flat)
    pool = G.zeros(sum(sizes), np.uint16)
    ptrs, offs, cnts = G.table(G.pool_tensors(fd, sizes, off))
    gf.call("gf_pack", F16, pool.data_ptr(), ptrs, offs, cnts, len(sizes), 1024.0, None)
    G.sync()
    assert (G.host(pool, np.uint16) == oracle.pack(flat, sizes, dtype=F16, scale=1024.0)).all()


def test_pack_errors(gf, G):
    with pytest.raises(gf.ConfigError):
        gf.call("gf_pack", 7, None, None, None, None, 0, 1.0, None)


# ---- K4 ring (colocated emulation: all ranks' buffers on one device) ---------------------------
def _ring_colocated(gf, G, bufs_np, dtype, windows=None, ring=None):
    bufs = [G.dev(b) for b in bufs_np]
    n = len(bufs)
    if windows is None:
        windows = (np.array([0], np.uint64), np.array([bufs_np[0].size], np.uint64))
    ws, wl = windows
    gf.call("gf_ring_allreduce_colocated", dtype, gf.ptr_array(bufs), n,
            None if ring is None else gf.int_array(ring), gf.u64_array(ws), gf.u64_array(wl),
            len(ws), None)
    G.sync()
    return [G.host(b, bufs_np[0].dtype) for b in bufs]


def test_ring_colocated_vs_dense_golden(gf, golden, oracle, G):
    g = golden("dense_sync.npz")
    for ci in range(int(g["dense_cases"][0])):
        p = f"d{ci}_"
        n, dt, theta = (int(x) for x in g[p + "meta"])
        sizes = g[p + "sizes"]
        ws, wl = oracle.dense_windows(sizes, 2 if dt == F16 else 4, theta)
        pools = [oracle.pack(gr, sizes, dtype=dt) for gr in g[p + "grads"]]
        out = _ring_colocated(gf, G, pools, dt, (ws, wl))
        for r in range(n):
            assert (G.bits(out[r]) == G.bits(g[p + "pools"][r])).all(), (ci, r)


@pytest.mark.parametrize("n", [2, 3, 4, 5, 8, 11, 16])
@pytest.mark.parametrize("dtype", [F16, F32])
def test_ring_colocated_random(gf, oracle, G, n, dtype):
    rng = np.random.default_rng(n * 10 + dtype)
    for L in (1, 7, 8, 97, 4099, 100003, 1 << 20):
        vals = [G.specials(rng, L) * np.float32(100) for _ in range(n)]
        bufs = [oracle.f2h(v) if dtype == F16 else v for v in vals]
        ring = rng.permutation(n)
        want = oracle.ring_allreduce([b.copy() for b in bufs], dtype=dtype, ring_order=ring)
        got = _ring_colocated(gf, G, bufs, dtype, ring=ring)
        for r in range(n):
            assert (G.bits(got[r]) == G.bits(want[r])).all(), (L, r)


def test_ring_colocated_resnet_windows(gf, oracle, G):
    """ResNet-50 gradient set, fp16, theta = 1 MiB windows (one launch), N=8."""
    n = 8
    off, _, _ = oracle.pool_layout(RESNET50, 32000)
    pools = [oracle.pack(oracle.gen_grads(100 + r, RESNET50), RESNET50, dtype=F16) for r in range(n)]
    ws, wl = oracle.dense_windows(RESNET50, 2, 1 << 20)
    want = oracle.ring_allreduce([p.copy() for p in pools], dtype=F16, windows=(ws, wl))
    got = _ring_colocated(gf, G, pools, F16, (ws, wl))
    for r in range(n):
        assert (got[r] == want[r]).all()


def test_ring_traffic_matches_reference_law(gf):
    # test_collectives.cpp:73-100: 2(N-1)K/N exact; N=4, K=1 KiB -> 1536 B
    for n in (2, 4, 8):
        for kb in (4 << 10, 1 << 20):
            s, r, f = C.c_uint64(), C.c_uint64(), C.c_uint64()
            gf.call("gf_ring_traffic", kb // 4, n, 0, F32, C.byref(s), C.byref(r), C.byref(f))
            assert s.value == 2 * (n - 1) * kb // n
    s, r, f = C.c_uint64(), C.c_uint64(), C.c_uint64()
    gf.call("gf_ring_traffic", 256, 4, 1, F32, C.byref(s), C.byref(r), C.byref(f))
    assert s.value == 1536 and f.value == 6


# ---- CSC kernels ------------------------------------------------------------------------------
@pytest.mark.parametrize("dtype", [F16, F32])
def test_chunk_norms(gf, oracle, G, dtype):
    rng = np.random.default_rng(21 + dtype)
    for total, chunk in ((61100840 if dtype == F16 else 3_000_000, 32000), (1000, 7), (5, 100)):
        x = rng.uniform(-1, 1, total).astype(np.float32)
        x[: min(total, 50000)] *= np.float32(60000)  # first chunks: huge -> exact fp64 fallback
        pool = oracle.f2h(x) if dtype == F16 else x
        off, nc, _ = oracle.pool_layout([total], chunk)
        imp = (rng.random(nc) < 0.3).astype(np.uint8)
        want = oracle.chunk_norms(pool, chunk, nc, imp, 3, dtype=dtype)
        out = G.zeros(nc, np.float32)
        pd, idev = G.dev(pool), G.dev(imp)
        gf.call("gf_chunk_norms", dtype, pd.data_ptr(), total, chunk, nc,
                idev.data_ptr(), 3, out.data_ptr(), None)
        G.sync()
        assert (G.bits(G.host(out)) == G.bits(want)).all(), (total, chunk)


def test_chunk_norms_nan(gf, oracle, G):
    x = np.ones(10000, np.float32)
    x[1234] = np.nan
    pool = oracle.f2h(x)
    want = oracle.chunk_norms(pool, 1000, 10, None, 1)
    out = G.zeros(10, np.float32)
    pd = G.dev(pool)
    gf.call("gf_chunk_norms", F16, pd.data_ptr(), 10000, 1000, 10, None, 1,
            out.data_ptr(), None)
    G.sync()
    assert (G.bits(G.host(out)) == G.bits(want)).all()


@pytest.mark.parametrize("dtype", [F16, F32])
def test_csc_correct_and_fused(gf, oracle, G, dtype):
    rng = np.random.default_rng(5)
    sizes = [300, 57, 1000, 8, 64000, 13]
    chunk = 96
    total = sum(sizes)
    off, nc, _ = oracle.pool_layout(sizes, chunk)
    flat = G.specials(rng, total, nan=False) * np.float32(2)
    hg0 = (rng.uniform(-1, 1, total) * 0.1).astype(np.float32)
    imp = (rng.random(nc) < 0.4).astype(np.uint8)
    mom = np.float32(0.9)
    # oracle: pack, correct, compact
    pool_w = oracle.pack(flat, sizes, dtype=dtype)
    hg_w = hg0.copy()
    oracle.csc_correct(pool_w, hg_w, imp, chunk, mom, dtype=dtype)
    stage_w = oracle.csc_compact(pool_w, imp, chunk, dtype=dtype)
    et = np.uint16 if dtype == F16 else np.float32
    # (a) in-place correction over a chunk range split in two calls
    pool_d = G.dev(oracle.pack(flat, sizes, dtype=dtype))
    hg_d, imp_d = G.dev(hg0), G.dev(imp)
    gf.call("gf_csc_correct", dtype, pool_d.data_ptr(), hg_d.data_ptr(), imp_d.data_ptr(), total,
            chunk, nc, 0, nc // 2, mom, None)
    gf.call("gf_csc_correct", dtype, pool_d.data_ptr(), hg_d.data_ptr(), imp_d.data_ptr(), total,
            chunk, nc, nc // 2, nc - nc // 2, mom, None)
    G.sync()
    assert (G.bits(G.host(pool_d, et)) == G.bits(pool_w)).all()
    assert (G.bits(G.host(hg_d)) == G.bits(hg_w)).all()
    # (b) plan + fused pack/correct/compact
    coff = G.zeros(nc, np.uint64)
    plan = G.zeros(4 + nc, np.uint64)
    gf.call("gf_csc_plan", imp_d.data_ptr(), total, chunk, nc, dtype, THETA_INF,
            coff.data_ptr(), plan.data_ptr(), None)
    fd = G.dev(flat)
    pool2 = G.zeros(total, et)
    hg2 = G.dev(hg0)
    stage = G.zeros(total, et)
    nacc = G.zeros(nc, np.uint64)
    ptrs, offs, cnts = G.table(G.pool_tensors(fd, sizes, off))
    gf.call("gf_csc_pack_correct", dtype, pool2.data_ptr(), hg2.data_ptr(), stage.data_ptr(),
            imp_d.data_ptr(), coff.data_ptr(), total, chunk, nc, ptrs, offs, cnts, len(sizes),
            mom, nacc.data_ptr() if dtype == F16 else None, None)
    G.sync()
    if dtype == F16:  # K3 fused into K2: exact L1 of every unimportant chunk
        want_l1 = oracle.chunk_norms(pool_w, chunk, nc, None, 1, dtype=dtype)
        got_u = G.host(nacc, np.uint64)
        for c in np.nonzero(imp == 0)[0]:
            assert np.float32(float(got_u[c]) * 2.0 ** -24) == want_l1[c], c
        assert not got_u[imp == 1].any()
    pl = G.host(plan, np.uint64)
    assert int(pl[0]) == stage_w.size and int(pl[1]) == int(imp.sum())
    assert (G.bits(G.host(pool2, et)) == G.bits(pool_w)).all()
    assert (G.bits(G.host(hg2)) == G.bits(hg_w)).all()
    assert (G.bits(G.host(stage, et)[: stage_w.size]) == G.bits(stage_w)).all()
    # (c) stand-alone compact and scatter round trip
    stage3 = G.zeros(total, et)
    gf.call("gf_csc_compact", dtype, pool2.data_ptr(), stage3.data_ptr(), plan.data_ptr(),
            coff.data_ptr(), total, chunk, nc, nc, None)
    G.sync()
    assert (G.bits(G.host(stage3, et)[: stage_w.size]) == G.bits(stage_w)).all()
    pool3 = G.zeros(total, et)
    gf.call("gf_csc_scatter", dtype, pool3.data_ptr(), stage3.data_ptr(), plan.data_ptr(),
            coff.data_ptr(), total, chunk, nc, nc, None, None)
    G.sync()
    want3 = np.zeros(total, et)
    oracle.csc_scatter(want3, imp, chunk, stage_w, dtype=dtype)
    assert (G.bits(G.host(pool3, et)) == G.bits(want3)).all()


def test_select_topk_and_plan(gf, oracle, G):
    rng = np.random.default_rng(8)
    for nc, k in ((4, 2), (3, 1), (1909, 191), (799, 80), (5000, 1), (3000, 3000), (2048, 1024),
                  (4096, 409), (4097, 409), (6000, 2999)):
        for kind in ("random", "ties", "zeros", "signed_zero_inf"):
            if kind == "random":
                norms = rng.uniform(0, 10, nc).astype(np.float32)
            elif kind == "ties":
                norms = rng.integers(0, 4, nc).astype(np.float32)
            elif kind == "signed_zero_inf":
                norms = rng.choice(np.array([0.0, -0.0, 1.5, np.inf, 3e38], np.float32), nc)
            else:
                norms = np.zeros(nc, np.float32)
            want = oracle.select_topk(norms, k)
            flags = G.zeros(nc, np.uint8)
            nd = G.dev(norms)
            gf.call("gf_select_topk", nd.data_ptr(), nc, k, flags.data_ptr(), None)
            G.sync()
            got = G.host(flags)
            assert (got == want).all(), (nc, k, kind)
            for theta in (0, 1000, 64000 * 3, THETA_INF):
                total = nc * 32 + 17
                coff = G.zeros(nc, np.uint64)
                plan = G.zeros(4 + nc, np.uint64)
                gf.call("gf_csc_plan", flags.data_ptr(), total, 32, nc, F16, theta,
                        coff.data_ptr(), plan.data_ptr(), None)
                G.sync()
                pl = G.host(plan, np.uint64).astype(np.int64)
                ws, wl = oracle.csc_windows(want, total, 32, 2, theta)
                staged, kc, nwin, stride = (int(v) for v in pl[:4])
                assert list(pl[4:4 + kc]) == list(np.nonzero(want)[0])
                assert nwin == len(ws)
                dev_w = [(w * stride, (staged - w * stride) if w == nwin - 1 else stride)
                         for w in range(nwin)]
                assert dev_w == list(zip(ws.tolist(), wl.tolist()))
                lens = np.where(np.arange(nc) == nc - 1, total - (nc - 1) * 32, 32) * want
                assert (G.host(coff, np.uint64) == np.concatenate([[0], np.cumsum(lens)[:-1]])).all()


def test_select_colocated_norm_exchange(gf, oracle, G):
    rng = np.random.default_rng(12)
    for n in (2, 3, 8):
        nc = 1909
        norms = [rng.uniform(0, 5, nc).astype(np.float32) for _ in range(n)]
        norms[0][:10] = 1.0  # ties
        for r in range(1, n):
            norms[r][:10] = 1.0
        want_sum = oracle.ring_allreduce([x.copy() for x in norms], dtype=F32)
        want = oracle.select_topk(want_sum[0], 191)
        dn = [G.dev(x) for x in norms]
        flags = G.zeros(nc, np.uint8)
        coff = G.zeros(nc, np.uint64)
        plan = G.zeros(4 + nc, np.uint64)
        gf.call("gf_csc_select_colocated", gf.ptr_array(dn), n, None, nc, 191, flags.data_ptr(),
                nc * 32000, 32000, F16, THETA_INF, coff.data_ptr(), plan.data_ptr(), None, None,
                None, None)
        G.sync()
        assert (G.host(flags) == want).all()
        for r in range(n):
            assert (G.bits(G.host(dn[r])) == G.bits(want_sum[0])).all()


@pytest.mark.parametrize("dtype", [F16, F32])
def test_sgd_updates(gf, oracle, golden, G, dtype):
    g = golden("csc_run.npz")
    p = "c0_"
    n, dt, theta, chunk, T = (int(x) for x in g[p + "meta"])
    if dt != dtype:
        p = "c3_"
        n, dt, theta, chunk, T = (int(x) for x in g[p + "meta"])
    total = int(g[p + "sizes"].sum())
    nc = oracle.pool_layout(g[p + "sizes"], chunk)[1]
    coff = G.zeros(nc, np.uint64)
    plan = G.zeros(4 + nc, np.uint64)
    for r in range(n):
        hu = G.zeros(total, np.float32)
        w = G.dev(g[p + "w0"])
        for t in range(T):
            pool = G.dev(g[p + "pool_x"][t][r])
            impd = G.dev(g[p + "imp"][t][r])
            gf.call("gf_csc_plan", impd.data_ptr(), total, chunk, nc, dt, THETA_INF,
                    coff.data_ptr(), plan.data_ptr(), None)
            gf.call("gf_csc_sgd_update", dt, pool.data_ptr(), plan.data_ptr(), total, chunk, nc,
                    nc, n, np.float32(0.9), np.float32(0.01), hu.data_ptr(), w.data_ptr(), None)
            G.sync()
            assert (G.bits(G.host(hu)) == G.bits(g[p + "hu"][t][r])).all()
            assert (G.bits(G.host(w)) == G.bits(g[p + "w"][t][r])).all()
    # dense update == csc update with every chunk important
    pool = G.dev(g[p + "pool_x"][0][0])
    hu1, w1 = G.zeros(total, np.float32), G.dev(g[p + "w0"])
    hu2, w2 = G.zeros(total, np.float32), G.dev(g[p + "w0"])
    ones = G.dev(np.ones(nc, np.uint8))
    gf.call("gf_csc_plan", ones.data_ptr(), total, chunk, nc, dt, THETA_INF, coff.data_ptr(),
            plan.data_ptr(), None)
    gf.call("gf_dense_sgd_update", dt, pool.data_ptr(), total, n, np.float32(0.9),
            np.float32(0.01), hu1.data_ptr(), w1.data_ptr(), None)
    gf.call("gf_csc_sgd_update", dt, pool.data_ptr(), plan.data_ptr(), total, chunk, nc, nc, n,
            np.float32(0.9), np.float32(0.01), hu2.data_ptr(), w2.data_ptr(), None)
    G.sync()
    assert (G.bits(G.host(w1)) == G.bits(G.host(w2))).all()


# ---- whole CSC iterations, colocated ranks, vs the reference's own multi-step run -------------
@pytest.mark.parametrize("fused_norms", [True, False])
def test_csc_multistep_colocated_vs_reference_golden(gf, golden, oracle, G, fused_norms):
    """Full CSC iterations (pack+correct+compact, ring, write-back, norms, exchange+top-k)
    for n colocated ranks against the reference's own multi-step run. fused_norms: exact
    chunk L1 accumulated inside pack_correct/scatter (fp16) instead of gf_chunk_norms."""
    g = golden("csc_run.npz")
    for ci in range(int(g["csc_cases"][0])):
        p = f"c{ci}_"
        n, dt, theta, chunk, T = (int(x) for x in g[p + "meta"])
        if fused_norms and dt != F16:
            continue
        sizes = [int(s) for s in g[p + "sizes"]]
        total = sum(sizes)
        off, nc, _ = oracle.pool_layout(sizes, chunk)
        et = np.uint16 if dt == F16 else np.float32
        pools = [G.zeros(total, et) for _ in range(n)]
        stages = [G.zeros(total, et) for _ in range(n)]
        hgs = [G.zeros(total, np.float32) for _ in range(n)]
        norms = [G.zeros(nc, np.float32) for _ in range(n)]
        naccs = [G.zeros(nc, np.uint64) for _ in range(n)] if fused_norms else None
        imp = G.dev(np.ones(nc, np.uint8))
        coff = G.zeros(nc, np.uint64)
        plan = G.zeros(4 + nc, np.uint64)
        gf.call("gf_csc_plan", imp.data_ptr(), total, chunk, nc, dt, theta, coff.data_ptr(),
                plan.data_ptr(), None)
        for t in range(T):
            for r in range(n):
                fd = G.dev(g[p + "grads"][t][r])
                ptrs, offs, cnts = G.table(G.pool_tensors(fd, sizes, off))
                gf.call("gf_csc_pack_correct", dt, pools[r].data_ptr(), hgs[r].data_ptr(),
                        stages[r].data_ptr(), imp.data_ptr(), coff.data_ptr(), total, chunk, nc,
                        ptrs, offs, cnts, len(sizes), np.float32(0.9),
                        naccs[r].data_ptr() if fused_norms else None, None)
                G.sync()
            gf.call("gf_ring_allreduce_colocated_planned", dt, gf.ptr_array(stages), n, None,
                    plan.data_ptr(), None)
            for r in range(n):
                gf.call("gf_csc_scatter", dt, pools[r].data_ptr(), stages[r].data_ptr(),
                        plan.data_ptr(), coff.data_ptr(), total, chunk, nc, nc,
                        naccs[r].data_ptr() if fused_norms else None, None)
                if not fused_norms:
                    gf.call("gf_chunk_norms", dt, pools[r].data_ptr(), total, chunk, nc,
                            imp.data_ptr(), n, norms[r].data_ptr(), None)
            k = oracle.selection_count(oracle.sparsity_at(t + 1, 2, 0.75), nc)
            nxt = G.zeros(nc, np.uint8)
            nxt_plan = G.zeros(4 + nc, np.uint64)
            nxt_coff = G.zeros(nc, np.uint64)
            gf.call("gf_csc_select_colocated", gf.ptr_array(norms), n, None, nc, k,
                    nxt.data_ptr(), total, chunk, dt, theta, nxt_coff.data_ptr(), nxt_plan.data_ptr(),
                    gf.ptr_array(naccs) if fused_norms else None,
                    gf.ptr_array(pools) if fused_norms else None,
                    imp.data_ptr() if fused_norms else None, None)
            G.sync()
            for r in range(n):
                assert (G.bits(G.host(hgs[r])) == G.bits(g[p + "hg"][t][r])).all(), (ci, t, r)
                assert (G.bits(G.host(pools[r], et)) == G.bits(g[p + "pool_x"][t][r])).all(), (ci, t, r)
                assert (G.bits(G.host(norms[r])) == G.bits(g[p + "norms_sum"][t][r])).all(), (ci, t, r)
                if fused_norms:
                    assert not G.host(naccs[r], np.uint64).any()  # re-armed for the next step
            assert (G.host(nxt) == g[p + "next_imp"][t][0]).all(), (ci, t)
            imp, coff, plan = nxt, nxt_coff, nxt_plan


@pytest.mark.parametrize("dtype", [F16, F32])
@pytest.mark.parametrize("aligned", [True, False])
def test_sync_step_world1_one_pass(gf, oracle, G, dtype, aligned):
    """world == 1: gf_sync_step_dense packs and unpacks in ONE pass (pack_kernel<DstTable>).
    Pool and g_avg vs the oracle, with special values; aligned=False shifts every output
    tensor by one element so the scalar path runs too."""
    import torch
    from paper_1902_06855_b200 import cudart
    from paper_1902_06855_b200.engine import GradSync
    sizes = RESNET50[:30] + [13, 7, 40000]
    off, _, _ = oracle.pool_layout(sizes, 32000)
    bounds = np.concatenate([[0], np.cumsum(sizes)])
    sync = GradSync(sizes, dtype=dtype, theta=1 << 16)
    total = int(bounds[-1])
    esz = 2 if dtype == F16 else 4
    rng = np.random.default_rng(7 + dtype)
    for it in range(2):
        flat = G.specials(rng, total) * np.float32(8 ** it)
        g = torch.from_numpy(flat).cuda()
        shift = 0 if aligned else 1
        out = torch.full((total + 1,), -1.0, device="cuda")
        gp = [g[int(bounds[i]):int(bounds[i + 1])].data_ptr() for i in range(len(sizes))]
        op = [out[shift + int(bounds[i]):shift + int(bounds[i + 1])].data_ptr() for i in range(len(sizes))]
        sync.dense_step(gp, op)
        torch.cuda.synchronize()
        want_pool = oracle.pack(flat, sizes, dtype=dtype)
        want = oracle.unpack(want_pool, 1, dtype=dtype)
        pool = np.empty(total * esz, np.uint8)
        cudart.memcpy(pool.ctypes.data, sync.pool_ptr, total * esz)
        assert (pool.view(np.uint16 if dtype == F16 else np.uint32) == G.bits(want_pool)).all()
        got = out.cpu().numpy()[shift:shift + total]
        for i, s in enumerate(sizes):
            assert (got[int(bounds[i]):int(bounds[i + 1])].view(np.uint32) ==
                    want[int(off[i]):int(off[i]) + s].view(np.uint32)).all(), (it, i)
    sync.close()


@pytest.mark.parametrize("dtype", [F16, F32])
@pytest.mark.parametrize("theta", [400, THETA_INF])
def test_engine_csc_world1_vs_oracle(gf, oracle, G, dtype, theta):
    """GradSync.csc_step at world 1 (the bench's N=1 CSC path: pack_correct, scatter,
    select beside the update on a second stream) over 5 iterations vs the oracle."""
    import torch
    from paper_1902_06855_b200 import cudart
    from paper_1902_06855_b200.engine import GradSync
    sizes, chunk = [300, 50, 1000, 7, 4000], 100
    total = sum(sizes)
    sync = GradSync(sizes, dtype=dtype, theta=theta, chunk=chunk, csc=True, final_sparsity=0.75,
                    warmup_iters=2, momentum=0.9, lr=0.01)
    nc = sync.layout.num_chunks
    rng = np.random.default_rng(5 + dtype)
    w0 = rng.uniform(-1, 1, total).astype(np.float32)
    wp, _ = sync.state("w")
    cudart.memcpy(wp, w0.ctypes.data, w0.nbytes)
    cudart.sync_device()

    def st(name, dt):
        p, n = sync.state(name)
        out = np.empty(n // np.dtype(dt).itemsize, dt)
        cudart.memcpy(out.ctypes.data, p, out.nbytes)
        cudart.sync_device()
        return out
    bounds = np.concatenate([[0], np.cumsum(sizes)])
    o_hg, o_hu, o_w = [np.zeros(total, np.float32)], np.zeros(total, np.float32), w0.copy()
    o_imp = np.ones(nc, np.uint8)
    esz = 2 if dtype == F16 else 4
    for t in range(5):
        x = G.specials(rng, total, nan=False) * np.float32(rng.uniform(0.1, 3))
        xd = torch.from_numpy(x).cuda()
        sync.csc_step([xd[int(bounds[i]):int(bounds[i + 1])].data_ptr() for i in range(len(sizes))])
        torch.cuda.synchronize()
        k = oracle.selection_count(oracle.sparsity_at(t + 1, 2, 0.75), nc)
        pools, _, nxt, _ = oracle.csc_iteration([x], sizes, chunk, theta, np.float32(0.9), o_imp, k, o_hg,
                                                dtype=dtype)
        oracle.csc_sgd_update(pools[0], o_imp, chunk, 1, np.float32(0.9), np.float32(0.01), o_hu, o_w,
                              dtype=dtype)
        assert (st("pool", np.uint8) == pools[0].view(np.uint8)).all(), t
        assert (G.bits(st("hg", np.float32)) == G.bits(o_hg[0])).all(), t
        assert (st("imp_next", np.uint8) == nxt).all(), t
        assert (G.bits(st("hu", np.float32)) == G.bits(o_hu)).all(), t
        assert (G.bits(st("w", np.float32)) == G.bits(o_w)).all(), t
        o_imp = nxt
    sync.close()


def test_overlap_api_world1(gf, oracle, G):
    """begin_iteration / tensor_complete / finalize_iteration at world 1: each closed theta
    window is packed and unpacked on the communication stream; out-of-order completion and
    an early finalize raise ConfigError like the reference (fusion.cpp:90-94)."""
    import torch
    from paper_1902_06855_b200 import capi
    from paper_1902_06855_b200.engine import GradSync
    sizes = RESNET50[:60] + [13, 7]
    off, _, _ = oracle.pool_layout(sizes, 32000)
    bounds = np.concatenate([[0], np.cumsum(sizes)])
    sync = GradSync(sizes, theta=1 << 18)
    flat = oracle.gen_grads(99, sizes)
    g = torch.from_numpy(flat).cuda()
    out = torch.empty_like(g)
    gp = [g[int(bounds[i]):int(bounds[i + 1])].data_ptr() for i in range(len(sizes))]
    op = [out[int(bounds[i]):int(bounds[i + 1])].data_ptr() for i in range(len(sizes))]
    sync.begin_iteration(gp, op)
    with pytest.raises(capi.ConfigError):
        sync.tensor_complete(1)
    for tid in range(len(sizes), 0, -1):
        sync.tensor_complete(tid)
    sync.finalize_iteration()
    torch.cuda.synchronize()
    want = oracle.unpack(oracle.pack(flat, sizes), 1)
    got = out.cpu().numpy()
    for i, s in enumerate(sizes):
        assert (got[int(bounds[i]):int(bounds[i + 1])].view(np.uint32) ==
                want[int(off[i]):int(off[i]) + s].view(np.uint32)).all(), i
    sync.begin_iteration(gp, op)
    sync.tensor_complete(len(sizes))
    with pytest.raises(capi.ConfigError):
        sync.finalize_iteration()
    sync.close()


def test_chunk_norms_every_finite_half(gf, oracle, G):
    """Exact-unit L1 (|h| * 2^24 via fp32, gf_device.cuh units8/half_units) over every finite
    half, one per chunk and eight per chunk, vs the oracle's sequential fp64 chunk_l1."""
    h = np.arange(65536, dtype=np.uint32).astype(np.uint16)
    h = h[(h & 0x7C00) != 0x7C00]
    for chunk in (1, 8):
        n = (h.size // chunk) * chunk
        pool = np.ascontiguousarray(h[:n])
        nc = n // chunk
        d = G.dev(pool)
        out = G.zeros(nc, np.float32)
        gf.call("gf_chunk_norms", F16, d.data_ptr(), n, chunk, nc, None, 1, out.data_ptr(), None)
        G.sync()
        want = oracle.chunk_norms(pool, chunk, nc, None, 1, dtype=F16)
        assert (G.bits(G.host(out)) == G.bits(want)).all(), chunk

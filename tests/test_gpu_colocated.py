# SPDX-License-Identifier: Apache-2.0
"""The multi-GPU path proven on ONE B200: N-rank worlds colocated on one device
(gf_comm_connect_colocated, tests/colo.py) run the default N>1 kernels exactly as across GPUs —
the routed pack + rsp_kernel (rspush), the pull RS/AG fused with the unpack, the push-pull
ring, both CSC exchange forms with their fused write-back, the inbox norm exchange of the
selection, the cross-rank flag/epoch protocol and its timeout — checked bit for bit against
the oracle and, at the BASELINE configs' full sizes, against the unmodified reference
(oracle/_ref) on the same seeded gradients.

References (paths relative to /root/reference/proj): ring sums and order
src/collectives.cpp:55-97; write-back src/sparse.cpp:162-168; fp32 norm allreduce
src/sparse.cpp:185-187; selection src/sparse.cpp:189-201; dense update read
src/trainer.cpp:336-342.
"""
import ctypes as C

import numpy as np
import pytest

from colo import ColoWorld, close_raw, raw_comms, read, to_dev, write

pytestmark = [pytest.mark.gpu]

F16, F32 = 1, 0
THETA_INF = (1 << 64) - 1
RAGGED = [5, 97, 1, 4099, 300_001, 8, 77, 3]  # total = 8k + 3: unaligned inbox slots (ADVICE)
assert sum(RAGGED) % 8 == 3


def many_sizes():
    rng = np.random.default_rng(3)
    s = rng.integers(1, 3000, 300).tolist()  # > 256 tensors (more than one launch table)
    s[-1] += (3 - sum(s) % 8) % 8 + 8
    return s


def bits(a):
    return a.view(np.uint16) if a.itemsize == 2 else a.view(np.uint32)


def flat_from_pool(pool_arr, offs, sizes):
    """Pool-ordered array -> flat ascending-id array."""
    return np.concatenate([pool_arr[int(o):int(o) + int(s)] for o, s in zip(offs, sizes)])


def grads_for(o, sizes, world, seed, specials=True):
    gs = []
    for r in range(world):
        g = o.gen_grads(seed * 131 + r, sizes)
        if specials:
            g[::97] *= 3e4       # clamped / overflowing sums
            g[5::1009] = np.nan  # NaN operands (x86 NaN rules in the sums)
            g[7::2003] = -np.inf
        gs.append(g)
    return gs


def check_dense(o, W, sizes, dtype, theta, grads, pools_got, outs_got, ring=None):
    esz = 2 if dtype == F16 else 4
    off, _, _ = o.pool_layout(sizes, 32000)
    ws, wl = o.dense_windows(sizes, esz, theta)
    pools = [o.pack(g, sizes, dtype=dtype) for g in grads]
    o.ring_allreduce(pools, dtype=dtype, windows=(ws, wl), ring_order=ring)
    for r in range(W):
        assert (bits(pools_got[r]) == bits(pools[r])).all(), ("pool", r)
        want = flat_from_pool(o.unpack(pools[r], W, dtype=dtype), off, sizes)
        assert (want.view(np.uint32) == outs_got[r].view(np.uint32)).all(), ("g_avg", r)


@pytest.mark.parametrize("world", [2, 3, 4, 8])
@pytest.mark.parametrize("mode,dtype", [("rspush", F16), ("pull", F16), ("push", F16), ("pull", F32),
                                        ("push", F32)])
@pytest.mark.parametrize("case", ["ragged", "many"])
def test_colo_dense_modes(oracle, world, mode, dtype, case):
    """Every dense N>1 exchange, three iterations with fresh data (pool / inbox reuse under the
    epoch protocol), theta windows from one per tensor to one for all, NaN/inf/overflow."""
    import torch
    sizes = RAGGED if case == "ragged" else many_sizes()
    thetas = [THETA_INF, 4096, 0] if case == "ragged" else [1 << 12]
    total = sum(sizes)
    for theta in thetas:
        cw = ColoWorld(world, sizes, dtype=dtype, theta=theta, dense_mode=mode)
        fallback = {"pull": "push"}  # beyond one 256-tensor table
        assert cw.ranks[0].dense_mode == (mode if len(sizes) <= 256 else fallback.get(mode, mode))
        try:
            for it in range(3):
                grads = grads_for(oracle, sizes, world, 10 * it + world)
                gd = [to_dev(g) for g in grads]
                outs = [torch.full((total,), float("nan"), device="cuda") for _ in range(world)]
                torch.cuda.synchronize()
                cw.dense_step(gd, outs)
                pools = [cw.state(r, "pool", np.uint16 if dtype == F16 else np.float32) for r in range(world)]
                check_dense(oracle, world, sizes, dtype, theta, grads, pools, [x.cpu().numpy() for x in outs])
        finally:
            cw.close()


@pytest.mark.parametrize("world,mode", [(1, "auto"), (2, "auto"), (4, "auto"), (8, "auto"), (2, "push"), (4, "pull")])
def test_colo_resnet50_full_vs_reference(oracle, reference, world, mode):
    """BASELINE configs[1]: ResNet-50, all 161 tensors, dense fp16 lazy allreduce (theta 64 MiB
    = one window), through the default engine path (one-pass kernel at N=1, rspush at N>1),
    on SURVEY §8(d)'s mt19937_64 gradients: pools and g_avg bit-exact vs the reference."""
    import torch
    from oracle.oracle import RESNET50
    from paper_1902_06855_b200 import capi
    sizes = RESNET50
    grads = [capi.synth_grads(r, 0, sizes) for r in range(world)]
    assert (grads[0][:1000].view(np.uint32) == reference.gen_grads(0, 0, sizes)[:1000].view(np.uint32)).all()
    pools_ref, gavg_ref, wb, _ = reference.dense_sync(grads, sizes, dtype=F16, theta=64 << 20)
    off, _, _ = oracle.pool_layout(sizes, 32000)
    cw = ColoWorld(world, sizes, theta=64 << 20, dense_mode=mode)
    try:
        assert cw.ranks[0].info().nwin == len(wb) == 1
        gd = [to_dev(g) for g in grads]
        outs = [torch.empty(sum(sizes), device="cuda") for _ in range(world)]
        torch.cuda.synchronize()
        cw.dense_step(gd, outs)
        for r in range(world):
            assert (cw.state(r, "pool", np.uint16) == pools_ref[r]).all(), r
            want = flat_from_pool(gavg_ref[r], off, sizes)
            assert (outs[r].cpu().numpy().view(np.uint32) == want.view(np.uint32)).all(), r
    finally:
        cw.close()


@pytest.mark.parametrize("mode", ["rspush", "push"])
def test_colo_alexnet_4rank_full_vs_reference(oracle, reference, mode):
    """BASELINE configs[0]: the AlexNet gradient set (61.1M params, 16 tensors), fp16 lazy
    allreduce, theta = inf, 4 ranks — the reference's own oracle run — bit-exact."""
    import torch
    from oracle.oracle import ALEXNET
    from paper_1902_06855_b200 import capi
    sizes, world = ALEXNET, 4
    grads = [capi.synth_grads(r, 0, sizes) for r in range(world)]
    pools_ref, gavg_ref, wb, _ = reference.dense_sync(grads, sizes, dtype=F16, theta=THETA_INF)
    assert list(wb) == [sum(sizes) * 2]
    off, _, _ = oracle.pool_layout(sizes, 32000)
    cw = ColoWorld(world, sizes, theta=THETA_INF, dense_mode=mode)
    try:
        gd = [to_dev(g) for g in grads]
        outs = [torch.empty(sum(sizes), device="cuda") for _ in range(world)]
        torch.cuda.synchronize()
        cw.dense_step(gd, outs)
        for r in range(world):
            assert (cw.state(r, "pool", np.uint16) == pools_ref[r]).all(), r
            want = flat_from_pool(gavg_ref[r], off, sizes)
            assert (outs[r].cpu().numpy().view(np.uint32) == want.view(np.uint32)).all(), r
    finally:
        cw.close()


def run_csc_vs_reference(reference, sizes, world, chunk, theta, steps, csc_mode, sparsity=0.9, warmup=0,
                         full=False, dtype=F16):
    """The engine's CSC iterations vs the reference's SparseState run on identical gradients:
    the selected set of every step, and (every step, or the last at full size) pool, residual
    hg, norms (fp32 ring sums), hu and w — all bit for bit."""
    from paper_1902_06855_b200 import capi
    grads = [[capi.synth_grads(r, t, sizes) for r in range(world)] for t in range(steps)]
    last = steps - 1
    probe = (0, world - 1)

    def keep(key, t, r):
        if key in ("next_imp", "norms_sum"):
            return True
        return (not full or t == last) and r in probe and key in ("pool_x", "hg", "hu", "w")

    ref = reference.csc_run(grads, sizes, chunk, dtype=dtype, theta=theta, final_sparsity=sparsity,
                            warmup=warmup, keep=keep)
    cw = ColoWorld(world, sizes, dtype=dtype, theta=theta, chunk=chunk, csc=True, final_sparsity=sparsity,
                   warmup_iters=warmup, csc_mode=csc_mode)
    pd = np.uint16 if dtype == F16 else np.float32
    try:
        for t in range(steps):
            gd = [to_dev(g) for g in grads[t]]
            import torch
            torch.cuda.synchronize()
            cw.csc_step(gd)
            for r in range(world):
                nxt = cw.state(r, "imp_next", np.uint8)
                assert (nxt == ref["next_imp"][t][r]).all(), ("selected set", t, r)
                norms = cw.state(r, "norms", np.float32)
                assert (norms.view(np.uint32) == ref["norms_sum"][t][r].view(np.uint32)).all(), ("norms", t, r)
            if full and t != last:
                continue
            for r in probe:
                assert (bits(cw.state(r, "pool", pd)) == bits(ref["pool_x"][t][r])).all(), ("pool", t, r)
                for key in ("hg", "hu", "w"):
                    got = cw.state(r, key, np.float32)
                    assert (got.view(np.uint32) == ref[key][t][r].view(np.uint32)).all(), (key, t, r)
    finally:
        cw.close()


@pytest.mark.parametrize("world", [2, 3, 4, 8])
@pytest.mark.parametrize("csc_mode", ["push", "pull"])
@pytest.mark.parametrize("theta", [0, 5000, THETA_INF])
def test_colo_csc_engine_vs_reference(reference, world, csc_mode, theta):
    """CSC (Algorithm 1) at N ranks, 5 iterations with a warm-up ramp, chunk 1000 (ragged last
    chunk), theta from one window per selected chunk to one window."""
    sizes = [1000, 64, 3000, 5, 8192, 7777, 12000, 31, 2048, 4099]
    run_csc_vs_reference(reference, sizes, world, 1000, theta, 5, csc_mode, sparsity=0.75, warmup=2)


@pytest.mark.parametrize("world,want", [(2, "push"), (3, "push"), (4, "pull"), (8, "pull")])
def test_colo_csc_mode_auto_resolution(world, want):
    """csc_mode auto: the routed pull exchange from 4 ranks, the ring below."""
    cw = ColoWorld(world, RAGGED, csc=True)
    try:
        assert cw.ranks[0].csc_mode == want
    finally:
        cw.close()


def test_colo_routed_csc_config_errors():
    """gf_comm_set_csc_inbox / gf_csc_pack_correct_routed reject what would overrun the heap or
    the inbox slots (ConfigError, nothing launched), and the routed pack needs the inbox set."""
    import ctypes as C
    import torch
    from paper_1902_06855_b200 import capi
    heap = 1 << 20
    comms, bases, streams = raw_comms(2, heap)
    try:
        with pytest.raises(capi.ConfigError):  # slots past the heap
            capi.call("gf_comm_set_csc_inbox", comms[0], heap - 1024, 4096)
        with pytest.raises(capi.ConfigError):  # slot length not a multiple of 8
            capi.call("gf_comm_set_csc_inbox", comms[0], 0, 1001)
        g = torch.zeros(5000, device="cuda")
        hg = torch.zeros(5000, device="cuda")
        pool = torch.zeros(5000, dtype=torch.float16, device="cuda")
        plan = torch.zeros(8, dtype=torch.int64, device="cuda")
        args = lambda c: (c, pool.data_ptr(), hg.data_ptr(), 0, plan.data_ptr(), 1000,  # noqa: E731
                          (C.c_void_p * 1)(g.data_ptr()), capi.u64_array([0]), capi.u64_array([5000]), 1,
                          np.float32(0.9), streams[0])
        with pytest.raises(capi.ConfigError):  # no inbox configured
            capi.call("gf_csc_pack_correct_routed", *args(comms[0]))
        capi.call("gf_comm_set_csc_inbox", comms[0], 1 << 16, 4096)
        with pytest.raises(capi.ConfigError):  # a 5000-element pool does not fit 4096-element slots
            capi.call("gf_csc_pack_correct_routed", *args(comms[0]))
        capi.call("gf_comm_set_csc_inbox", comms[0], 2 ** 64 - 1, 0)  # switched back off
        with pytest.raises(capi.ConfigError):
            capi.call("gf_csc_pack_correct_routed", *args(comms[0]))
    finally:
        close_raw(comms, streams)


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("csc_mode", ["push", "pull"])
def test_colo_alexnet_csc_full_vs_reference(reference, world, csc_mode):
    """BASELINE configs[2]: AlexNet with CSC (chunk 32000, 1909 chunks, keep the top 10 % =
    k 191), residual carry-over over 3 iterations (step 0 dense, then sparse) — the selected
    chunk set of every step and the final pool / hg / hu / w bit-exact vs the reference."""
    from oracle.oracle import ALEXNET
    run_csc_vs_reference(reference, ALEXNET, world, 32000, THETA_INF, 3, csc_mode, full=True)


@pytest.mark.parametrize("world,csc_mode", [(4, "push"), (8, "pull")])
def test_colo_resnet50_csc_theta_full_vs_reference(reference, world, csc_mode):
    """BASELINE configs[3]: ResNet-50 CSC with a lazy-fusion threshold (1 MiB: many windows over
    the staging buffer) and residual carry-over, 3 iterations, at 4 and 8 ranks."""
    from oracle.oracle import RESNET50
    run_csc_vs_reference(reference, RESNET50, world, 32000, 1 << 20, 3, csc_mode, full=True)


def test_colo_overlap_windows(oracle):
    """begin_iteration / tensor_complete / finalize_iteration at N=2: each theta window packed,
    ring-reduced and unpacked on the communication stream as it closes (fusion.cpp:72-123)."""
    import torch
    from colo import tensor_table
    sizes, world, theta = RAGGED, 2, 4096
    cw = ColoWorld(world, sizes, theta=theta)
    try:
        for it in range(2):
            grads = grads_for(oracle, sizes, world, 40 + it)
            gd = [to_dev(g) for g in grads]
            outs = [torch.zeros(sum(sizes), device="cuda") for _ in range(world)]
            torch.cuda.synchronize()
            gt = [tensor_table(g, sizes) for g in gd]
            ot = [tensor_table(x, sizes) for x in outs]
            for r in range(world):
                cw.ranks[r].begin_iteration(gt[r], ot[r], stream=cw.streams[r])
            for tid in range(len(sizes), 0, -1):  # backward order; ranks interleave
                for r in range(world):
                    cw.ranks[r].tensor_complete(tid)
            cw.run(lambda r, g, s: g.finalize_iteration())
            pools = [cw.state(r, "pool", np.uint16) for r in range(world)]
            check_dense(oracle, world, sizes, F16, theta, grads, pools, [x.cpu().numpy() for x in outs])
    finally:
        cw.close()


@pytest.mark.parametrize("world", [2, 5])
def test_colo_ring_raw_bit_exact(oracle, world):
    """gf_ring_allreduce (push-pull ring_kernel, P2P instantiation) over the symmetric heaps:
    random lengths, both dtypes, a non-identity ring order, NaNs; then 40 back-to-back small
    collectives with fresh data (the epoch protocol under reuse)."""
    from paper_1902_06855_b200 import capi
    comms, bases, streams = raw_comms(world, 64 << 20)
    try:
        order = np.random.default_rng(7).permutation(world).astype(np.int32)
        for c in comms:
            capi.call("gf_comm_set_ring_order", c, capi.int_array(order))
        for L in (1, 5, 8, 97, 4099, 1 << 20, 3_000_001):
            for dt in (F16, F32):
                vals = []
                for r in range(world):
                    rr = np.random.default_rng(1000 * L + 10 * r + dt)
                    x = rr.uniform(-100, 100, L).astype(np.float32)
                    x[rr.random(L) < 0.001] = np.nan
                    vals.append(oracle.f2h(x) if dt == F16 else x)
                for r in range(world):
                    write(bases[r] + 4096, vals[r])
                for r in range(world):
                    capi.call("gf_ring_allreduce", comms[r], dt, 4096, capi.u64_array([0]), capi.u64_array([L]), 1,
                              streams[r])
                want = oracle.ring_allreduce([v.copy() for v in vals], dtype=dt, ring_order=order)
                for r in range(world):
                    got = read(bases[r] + 4096, vals[r].nbytes, vals[r].dtype, streams[r])
                    assert (bits(got) == bits(want[r])).all(), (L, dt, r)
        for it in range(40):
            vals = [np.random.default_rng(10_000 + 31 * it + r).uniform(-4, 4, 67).astype(np.float32)
                    for r in range(world)]
            for r in range(world):
                write(bases[r], vals[r])
            for r in range(world):
                capi.call("gf_ring_allreduce", comms[r], F32, 0, capi.u64_array([0]), capi.u64_array([67]), 1,
                          streams[r])
            want = oracle.ring_allreduce([v.copy() for v in vals], dtype=F32, ring_order=order)
            for r in range(world):
                assert (bits(read(bases[r], 268, np.float32, streams[r])) == bits(want[r])).all(), it
        for c in comms:
            capi.call("gf_comm_status", c)
    finally:
        close_raw(comms, streams)


@pytest.mark.parametrize("world", [2, 4])
def test_colo_csc_exchange_forms_many_windows(oracle, world):
    """The CSC exchange with its fused write-back over MANY planned windows (theta = 0: one
    window per selected chunk), push form (ring_kernel + wb_segment) and pull form
    (csc_pull_kernel): pool bits and the exact L1 units of the received chunks."""
    import torch
    from paper_1902_06855_b200 import capi
    chunk, nc = 1000, 700
    total = nc * chunk - 1000 + 1377
    comms, bases, streams = raw_comms(world, 8 << 20)
    rng = np.random.default_rng(5)
    try:
        for theta in (0, 2 * chunk * 2 + 1, 77 * chunk * 2, THETA_INF):
            for form in ("push", "pull"):
                imp = (rng.random(nc) < 0.3).astype(np.uint8)
                imp[-1] = 1
                impd = torch.from_numpy(imp).cuda()
                coff = torch.zeros(nc, dtype=torch.int64, device="cuda")
                plan = torch.zeros(4 + nc, dtype=torch.int64, device="cuda")
                capi.call("gf_csc_plan", impd.data_ptr(), total, chunk, nc, F16, theta, coff.data_ptr(),
                          plan.data_ptr(), None)
                torch.cuda.synchronize()
                staged = int(plan[0].item())
                stg = [oracle.f2h(np.random.default_rng(theta % 997 + 10 * r + (form == "pull"))
                                  .uniform(-2, 2, staged).astype(np.float32)) for r in range(world)]
                pool0 = [oracle.f2h(np.random.default_rng(77 + r).uniform(-1, 1, total).astype(np.float32))
                         for r in range(world)]
                pools = [to_dev(p.copy()) for p in pool0]
                naccs = [torch.zeros(nc, dtype=torch.int64, device="cuda") for _ in range(world)]
                for r in range(world):
                    write(bases[r], stg[r])
                torch.cuda.synchronize()
                for r in range(world):
                    if form == "push":
                        capi.call("gf_ring_allreduce_planned_scatter", comms[r], F16, 0, plan.data_ptr(),
                                  pools[r].data_ptr(), chunk, nc, naccs[r].data_ptr(), streams[r])
                    else:
                        capi.call("gf_csc_exchange_pull", comms[r], 0, plan.data_ptr(), pools[r].data_ptr(), chunk,
                                  nc, naccs[r].data_ptr(), streams[r])
                for s in streams:
                    capi_sync(s)
                ws, wl = oracle.csc_windows(imp, total, chunk, 2, theta)
                assert int(plan[2].item()) == len(ws)
                red = oracle.ring_allreduce([x.copy() for x in stg], dtype=F16, windows=(ws, wl))
                lens = np.where(np.arange(nc) == nc - 1, total - (nc - 1) * chunk, chunk)
                for r in range(world):
                    want = pool0[r].copy()
                    s0 = 0
                    units = np.zeros(nc, np.int64)
                    for c in np.nonzero(imp)[0]:
                        L = int(lens[c])
                        want[c * chunk:c * chunk + L] = red[r][s0:s0 + L]
                        units[c] = int((np.abs(oracle.h2f(red[r][s0:s0 + L]).astype(np.float64)) * 2.0 ** 24).sum())
                        s0 += L
                    assert (pools[r].cpu().numpy().view(np.uint16) == want).all(), (theta, form, r)
                    assert (naccs[r].cpu().numpy()[imp == 1] == units[imp == 1]).all(), (theta, form, r)
        for c in comms:
            capi.call("gf_comm_status", c)
    finally:
        close_raw(comms, streams)


def capi_sync(s):
    from paper_1902_06855_b200 import cudart
    cudart.stream_sync(s)


def test_colo_select_inbox(oracle):
    """gf_csc_select's push-inbox norm exchange at N=3 (one barrier): fp32 ring-order sums and
    the top-k (ties to the lower index) over several rounds."""
    import torch
    from paper_1902_06855_b200 import capi
    world, nc, k = 3, 1909, 191
    noff, ioff = 0, 1 << 20
    comms, bases, streams = raw_comms(world, 2 << 20)
    try:
        for c in comms:
            capi.call("gf_comm_set_select_inbox", c, ioff)
        flags = [torch.zeros(nc, dtype=torch.uint8, device="cuda") for _ in range(world)]
        coff = [torch.zeros(nc, dtype=torch.int64, device="cuda") for _ in range(world)]
        plan = [torch.zeros(4 + nc, dtype=torch.int64, device="cuda") for _ in range(world)]
        torch.cuda.synchronize()
        for it in range(4):
            norms = [np.random.default_rng(100 * it + r).uniform(0, 5, nc).astype(np.float32) for r in range(world)]
            for r in range(world):
                norms[r][: 16 * (it + 1)] = 1.25  # ties
                write(bases[r] + noff, norms[r])
            for r in range(world):
                capi.call("gf_csc_select", comms[r], noff, nc, k + it, flags[r].data_ptr(), nc * 32000, 32000, F16,
                          THETA_INF, coff[r].data_ptr(), plan[r].data_ptr(), None, None, None, streams[r])
            for s in streams:
                capi_sync(s)
            want_sum = oracle.ring_allreduce([x.copy() for x in norms], dtype=F32)
            for r in range(world):
                got = read(bases[r] + noff, nc * 4, np.float32)
                assert (bits(got) == bits(want_sum[r])).all(), (it, r)
                assert (flags[r].cpu().numpy() == oracle.select_topk(want_sum[0], k + it)).all(), (it, r)
    finally:
        close_raw(comms, streams)


def test_colo_timeout_is_transport_error():
    """A rank that never reaches the collective: the others' device-side barrier times out,
    the communicator is poisoned and every later call fails fast (inproc.cpp:28-36)."""
    from paper_1902_06855_b200 import capi
    comms, bases, streams = raw_comms(2, 1 << 20)
    try:
        capi.call("gf_comm_set_timeout_ms", comms[0], 500)
        capi.call("gf_ring_allreduce", comms[0], F32, 0, capi.u64_array([0]), capi.u64_array([1024]), 1, streams[0])
        capi_sync(streams[0])
        with pytest.raises(capi.TransportError):
            capi.call("gf_comm_status", comms[0])
        with pytest.raises(capi.TransportError):
            capi.call("gf_ring_allreduce", comms[0], F32, 0, capi.u64_array([0]), capi.u64_array([8]), 1, streams[0])
    finally:
        close_raw(comms, streams)


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("csc_mode", ["push", "pull"])
def test_colo_csc_exchange_small_ctas(reference, world, csc_mode, monkeypatch):
    """The CSC exchange with its grid capped and 256-thread CTAs (GF_CSC_XBLOCKS /
    GF_CSC_XTHREADS, the engine's overlap knobs): same results as the reference."""
    monkeypatch.setenv("GF_CSC_XBLOCKS", "8")
    monkeypatch.setenv("GF_CSC_XTHREADS", "256")
    sizes = [1000, 64, 3000, 5, 8192, 7777, 12000, 31, 2048, 4099]
    run_csc_vs_reference(reference, sizes, world, 1000, 3000, 4, csc_mode, sparsity=0.75, warmup=1)

# SPDX-License-Identifier: Apache-2.0
"""Multi-GPU parity of the NVLink peer-memory path (one process per GPU, IPC-mapped heaps,
exactly the bench's launch model), plus the in-process multi-device bootstrap.

Each worker builds every rank's inputs deterministically, so it can compute the oracle
result for the whole world locally and compare its own rank bit-for-bit.
"""
import ctypes as C
import os
import socket

import numpy as np
import pytest

pytestmark = [pytest.mark.gpu]

F16, F32 = 1, 0
HEAP = 256 << 20


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _setup(rank, world, port):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch
    import torch.distributed as dist
    from paper_1902_06855_b200 import capi, cudart
    torch.cuda.set_device(rank)
    cudart.set_device(rank)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    comm = C.c_void_p()
    capi.call("gf_comm_create", world, rank, rank, HEAP, C.byref(comm))
    h = (C.c_char * capi.GF_IPC_HANDLE_BYTES)()
    capi.call("gf_comm_export_handle", comm, h)
    hs = [None] * world
    dist.all_gather_object(hs, bytes(h))
    capi.call("gf_comm_connect_ipc", comm, b"".join(hs))
    base = C.c_void_p()
    capi.call("gf_comm_heap", comm, C.byref(base), None)
    return comm, base.value, capi, cudart, dist


def _put(cudart, base, off, arr):
    arr = np.ascontiguousarray(arr)
    cudart.memcpy(base + off, arr.ctypes.data, arr.nbytes)
    cudart.sync_device()


def _get(cudart, base, off, like):
    out = np.empty_like(like)
    cudart.memcpy(out.ctypes.data, base + off, out.nbytes)
    cudart.sync_device()
    return out


def _bits(a):
    return a.view(np.uint16) if a.itemsize == 2 else a.view(np.uint32)


def _worker_ring(rank, world, port):
    comm, base, capi, cudart, dist = _setup(rank, world, port)
    from oracle.oracle import RESNET50, Oracle
    o = Oracle()
    # (1) ResNet-50 fp16 pool, theta = 1 MiB windows (bit-exact vs the oracle ring)
    pools = [o.pack(o.gen_grads(50 + r, RESNET50), RESNET50, dtype=F16) for r in range(world)]
    ws, wl = o.dense_windows(RESNET50, 2, 1 << 20)
    _put(cudart, base, 0, pools[rank])
    capi.call("gf_ring_allreduce", comm, F16, 0, capi.u64_array(ws), capi.u64_array(wl), len(ws), None)
    got = _get(cudart, base, 0, pools[rank])
    want = o.ring_allreduce([p.copy() for p in pools], dtype=F16, windows=(ws, wl))
    assert (got == want[rank]).all(), "resnet windows"
    # (2) random lengths, both dtypes, a non-identity ring order, NaN-bearing data
    rng = np.random.default_rng(7)
    order = rng.permutation(world).astype(np.int32)
    capi.call("gf_comm_set_ring_order", comm, capi.int_array(order))
    for L in (1, 5, 8, 97, 4099, 1 << 20, 3_000_001):
        for dt in (F16, F32):
            vals = []
            for r in range(world):
                rr = np.random.default_rng(1000 * L + 10 * r + dt)
                x = rr.uniform(-100, 100, L).astype(np.float32)
                x[rr.random(L) < 0.001] = np.nan
                vals.append(o.f2h(x) if dt == F16 else x)
            _put(cudart, base, 4096, vals[rank])
            capi.call("gf_ring_allreduce", comm, dt, 4096, capi.u64_array([0]), capi.u64_array([L]),
                      1, None)
            got = _get(cudart, base, 4096, vals[rank])
            want = o.ring_allreduce([v.copy() for v in vals], dtype=dt, ring_order=order)
            assert (_bits(got) == _bits(want[rank])).all(), (L, dt)
    # (3) back-to-back small collectives, fresh data each time (epoch protocol under reuse)
    capi.call("gf_comm_set_ring_order", comm, capi.int_array(range(world)))
    for it in range(60):
        vals = [np.random.default_rng(10_000 + 31 * it + r).uniform(-4, 4, 67).astype(np.float32)
                for r in range(world)]
        _put(cudart, base, 0, vals[rank])
        capi.call("gf_ring_allreduce", comm, F32, 0, capi.u64_array([0]), capi.u64_array([67]), 1, None)
        got = _get(cudart, base, 0, vals[rank])
        want = o.ring_allreduce([v.copy() for v in vals], dtype=F32)
        assert (_bits(got) == _bits(want[rank])).all(), it
    capi.call("gf_comm_status", comm)
    dist.barrier()


def _worker_rsag(rank, world, port):
    """gf_ring_allreduce_unpack (pull RS + pull AG fused with the unpack): pools and g_avg
    bit-exact vs the oracle ring + unpack, with and without the exit barrier."""
    comm, base, capi, cudart, dist = _setup(rank, world, port)
    import torch
    from oracle.oracle import RESNET50, Oracle
    o = Oracle()
    rng = np.random.default_rng(11)
    order = rng.permutation(world).astype(np.int32)
    cases = [(RESNET50, F16, 1 << 20), (RESNET50, F16, capi.THETA_INF),
             ([5, 97, 1, 4099, 3_000_001, 8, 77], F16, 4096), ([5, 97, 1, 4099, 300_001, 8, 77], F32, 1 << 16),
             ([3], F16, capi.THETA_INF), ([1, 2], F32, capi.THETA_INF)]
    it = 0
    for ci, (sizes, dt, theta) in enumerate(cases):
        esz = 2 if dt == F16 else 4
        off, _, _ = o.pool_layout(sizes, 32000)
        ws, wl = o.dense_windows(sizes, esz, theta)
        total = int(sum(sizes))
        pool_offs = [0, ((total * esz + 4095) // 4096) * 4096]
        cur = order if ci % 2 else np.arange(world, dtype=np.int32)
        capi.call("gf_comm_set_ring_order", comm, capi.int_array(cur))
        for flags in (0, capi.GF_RSAG_NO_EXIT_BARRIER):
            for rep in range(3):  # fresh data each time: pool reuse under both protocols
                it += 1
                grads = [o.gen_grads(100 * it + r, sizes) for r in range(world)]
                for r in range(world):
                    grads[r][::97] *= 3e4  # clamped / overflowing sums
                pools = [o.pack(g, sizes, dtype=dt) for g in grads]
                po = pool_offs[rep % 2] if flags else 0
                _put(cudart, base, po, pools[rank])
                # dst: one flat fp32 buffer cut at odd offsets (unaligned tensors take the scalar path)
                flat = torch.full((total + 3,), float("nan"), device="cuda")
                bounds = np.concatenate([[0], np.cumsum(sizes)])
                shift = 1 if it % 2 else 0
                dst = [flat[shift + int(bounds[i]):shift + int(bounds[i + 1])].data_ptr() for i in range(len(sizes))]
                capi.call("gf_ring_allreduce_unpack", comm, dt, po, capi.ptr_array(dst), capi.u64_array(off),
                          capi.u64_array(sizes), len(sizes), capi.u64_array(ws), capi.u64_array(wl), len(ws),
                          flags, None)
                torch.cuda.synchronize()
                want = o.ring_allreduce([p.copy() for p in pools], dtype=dt, windows=(ws, wl), ring_order=cur)
                got_pool = _get(cudart, base, po, pools[rank])
                assert (_bits(got_pool) == _bits(want[rank])).all(), (sizes[:3], dt, theta, flags, rep)
                g_avg = o.unpack(want[rank], world, dtype=dt)
                h = flat.cpu().numpy()[shift:shift + total]
                for i, sz in enumerate(sizes):
                    a = h[int(bounds[i]):int(bounds[i + 1])]
                    b = g_avg[int(off[i]):int(off[i]) + sz]
                    assert (a.view(np.uint32) == b.view(np.uint32)).all(), ("g_avg", i, dt, flags)
    capi.call("gf_comm_status", comm)
    dist.barrier()


def _worker_csc_windows(rank, world, port):
    """The CSC exchange with its write-back over MANY planned windows (theta = 0: one window
    per selected chunk), push form (gf_ring_allreduce_planned_scatter) and pull form
    (gf_csc_exchange_pull): pool bits and exact L1 units of the received chunks vs the oracle."""
    comm, base, capi, cudart, dist = _setup(rank, world, port)
    import torch
    from oracle.oracle import Oracle
    o = Oracle()
    chunk, nc = 1000, 700
    total = nc * chunk - 1000 + 1377  # longer last chunk
    soff = 0
    rng = np.random.default_rng(5)
    for theta in (0, 2 * chunk * 2 + 1, 77 * chunk * 2, capi.THETA_INF):
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
            stg = [o.f2h(np.random.default_rng(1000 * theta % 997 + 10 * r + (form == "pull")).uniform(-2, 2, staged)
                         .astype(np.float32)) for r in range(world)]
            pool0 = o.f2h(np.random.default_rng(77 + rank).uniform(-1, 1, total).astype(np.float32))
            _put(cudart, base, soff, stg[rank])
            pool = torch.from_numpy(pool0.view(np.int16).copy()).cuda()
            nacc = torch.zeros(nc, dtype=torch.int64, device="cuda")
            if form == "push":
                capi.call("gf_ring_allreduce_planned_scatter", comm, F16, soff, plan.data_ptr(), pool.data_ptr(),
                          chunk, nc, nacc.data_ptr(), None)
            else:
                capi.call("gf_csc_exchange_pull", comm, soff, plan.data_ptr(), pool.data_ptr(), chunk, nc,
                          nacc.data_ptr(), None)
            torch.cuda.synchronize()
            capi.call("gf_comm_status", comm)
            ws, wl = o.csc_windows(imp, total, chunk, 2, theta)
            assert int(plan[2].item()) == len(ws)
            red = o.ring_allreduce([x.copy() for x in stg], dtype=F16, windows=(ws, wl))[rank]
            want = pool0.copy()
            lens = np.where(np.arange(nc) == nc - 1, total - (nc - 1) * chunk, chunk)
            s0 = 0
            want_units = np.zeros(nc, np.int64)
            for c in np.nonzero(imp)[0]:
                L = int(lens[c])
                want[c * chunk:c * chunk + L] = red[s0:s0 + L]
                f = np.abs(o.h2f(red[s0:s0 + L]).astype(np.float64))
                want_units[c] = int((f * 2.0 ** 24).sum())
                s0 += L
            got = pool.cpu().numpy().view(np.uint16)
            assert (got == want).all(), (theta, form)
            assert (nacc.cpu().numpy()[imp == 1] == want_units[imp == 1]).all(), (theta, form)
            dist.barrier()
    dist.barrier()


def _worker_csc(rank, world, port):
    comm, base, capi, cudart, dist = _setup(rank, world, port)
    from oracle.oracle import Oracle
    o = Oracle()
    import torch
    nc, k = 1909, 191
    norms = [np.random.default_rng(r).uniform(0, 5, nc).astype(np.float32) for r in range(world)]
    for r in range(world):
        norms[r][:32] = 2.5  # ties across the threshold region
    noff = 1 << 20
    _put(cudart, base, noff, norms[rank])
    flags = torch.zeros(nc, dtype=torch.uint8, device="cuda")
    coff = torch.zeros(nc, dtype=torch.int64, device="cuda")
    plan = torch.zeros(4 + nc, dtype=torch.int64, device="cuda")
    total = nc * 32000 + 12840
    capi.call("gf_csc_select", comm, noff, nc, k, flags.data_ptr(), total, 32000, F16,
              capi.THETA_INF, coff.data_ptr(), plan.data_ptr(), None, None, None, None)
    torch.cuda.synchronize()
    want_sum = o.ring_allreduce([x.copy() for x in norms], dtype=F32)
    got_sum = _get(cudart, base, noff, norms[rank])
    assert (_bits(got_sum) == _bits(want_sum[rank])).all()
    want = o.select_topk(want_sum[0], k)
    assert (flags.cpu().numpy() == want).all()
    # planned ring over a staging buffer laid out by the plan (CSC exchange path)
    staged = int(plan[0].item())
    stg = [o.f2h(np.random.default_rng(90 + r).uniform(-1, 1, staged).astype(np.float32))
           for r in range(world)]
    soff = 8 << 20
    _put(cudart, base, soff, stg[rank])
    capi.call("gf_ring_allreduce_planned", comm, F16, soff, plan.data_ptr(), None)
    got = _get(cudart, base, soff, stg[rank])
    wantr = o.ring_allreduce([s.copy() for s in stg], dtype=F16)
    assert (got == wantr[rank]).all()
    dist.barrier()
    # push-inbox norm exchange (one barrier): same sums and set, several rounds
    capi.call("gf_comm_set_select_inbox", comm, 2 << 20)
    for it in range(4):
        norms = [np.random.default_rng(100 * it + r).uniform(0, 5, nc).astype(np.float32) for r in range(world)]
        for r in range(world):
            norms[r][: 16 * (it + 1)] = 1.25  # ties
        _put(cudart, base, noff, norms[rank])
        capi.call("gf_csc_select", comm, noff, nc, k + it, flags.data_ptr(), total, 32000, F16,
                  capi.THETA_INF, coff.data_ptr(), plan.data_ptr(), None, None, None, None)
        torch.cuda.synchronize()
        capi.call("gf_comm_status", comm)
        want_sum = o.ring_allreduce([x.copy() for x in norms], dtype=F32)
        assert (_bits(_get(cudart, base, noff, norms[rank])) == _bits(want_sum[rank])).all(), it
        assert (flags.cpu().numpy() == o.select_topk(want_sum[0], k + it)).all(), it
        dist.barrier()  # the next round's pushes follow every rank's reads (the exchange's role)
    capi.call("gf_comm_set_select_inbox", comm, (1 << 64) - 1)
    dist.barrier()


def _worker_timeout(rank, world, port):
    comm, base, capi, cudart, dist = _setup(rank, world, port)
    capi.call("gf_comm_set_timeout_ms", comm, 1500)
    if rank == 0:
        capi.call("gf_ring_allreduce", comm, F32, 0, capi.u64_array([0]), capi.u64_array([1024]),
                  1, None)
        cudart.sync_device()
        with pytest.raises(capi.TransportError):
            capi.call("gf_comm_status", comm)
        with pytest.raises(capi.TransportError):  # poisoned: later collectives fail fast
            capi.call("gf_ring_allreduce", comm, F32, 0, capi.u64_array([0]), capi.u64_array([8]),
                      1, None)
    dist.barrier()


def _spawn(fn, world):
    import torch.multiprocessing as mp
    mp.spawn(fn, args=(world, _free_port()), nprocs=world, join=True)


def _world():
    import torch
    return min(torch.cuda.device_count(), 8)


@pytest.mark.multigpu(2)
def test_p2p_ring_bit_exact():
    _spawn(_worker_ring, _world())


@pytest.mark.multigpu(2)
def test_p2p_ring_allreduce_unpack_bit_exact():
    _spawn(_worker_rsag, _world())


@pytest.mark.multigpu(2)
def test_p2p_csc_exchange_many_windows():
    _spawn(_worker_csc_windows, _world())


@pytest.mark.multigpu(2)
def test_p2p_csc_select_and_planned_ring():
    _spawn(_worker_csc, _world())


@pytest.mark.multigpu(2)
def test_p2p_timeout_is_transport_error():
    _spawn(_worker_timeout, 2)


@pytest.mark.multigpu(2)
def test_inprocess_local_connect():
    """One process driving every GPU (the reference's ranks-as-threads model)."""
    import torch
    from oracle.oracle import Oracle
    from paper_1902_06855_b200 import capi, cudart
    o = Oracle()
    world = _world()
    comms = []
    for r in range(world):
        c = C.c_void_p()
        capi.call("gf_comm_create", world, r, r, 64 << 20, C.byref(c))
        comms.append(c)
    capi.call("gf_comm_connect_local", (C.c_void_p * world)(*[c.value for c in comms]), world)
    L = 1_000_003
    vals = [o.f2h(np.random.default_rng(r).uniform(-9, 9, L).astype(np.float32)) for r in range(world)]
    bases = []
    for r in range(world):
        b = C.c_void_p()
        capi.call("gf_comm_heap", comms[r], C.byref(b), None)
        bases.append(b.value)
        cudart.set_device(r)
        cudart.memcpy(b.value, vals[r].ctypes.data, vals[r].nbytes)
        cudart.sync_device()
    for r in range(world):  # asynchronous launches on every device from one thread
        cudart.set_device(r)
        capi.call("gf_ring_allreduce", comms[r], F16, 0, capi.u64_array([0]), capi.u64_array([L]), 1, None)
    want = o.ring_allreduce([v.copy() for v in vals], dtype=F16)
    for r in range(world):
        cudart.set_device(r)
        cudart.sync_device()
        out = np.empty_like(vals[r])
        cudart.memcpy(out.ctypes.data, bases[r], out.nbytes)
        cudart.sync_device()
        assert (out == want[r]).all()
    for c in comms:
        capi.call("gf_comm_destroy", c)
    torch.cuda.synchronize()


def _worker_fused(rank, world, port):
    """The engine's dense step in every mode — the routed pack + local reduce + push all-gather
    (rspush), pack + pull RS/AG with the unpack fused in (alternating pools), pack + push-pull
    ring + unpack — over several iterations and theta values, bit-exact vs the oracle."""
    comm, base, capi, cudart, dist = _setup(rank, world, port)
    import torch
    from oracle.oracle import RESNET50, Oracle
    from paper_1902_06855_b200.engine import GradSync
    o = Oracle()
    torch.cuda.set_device(rank)
    sizes = RESNET50
    off, _, _ = o.pool_layout(sizes, 32000)
    bounds = np.concatenate([[0], np.cumsum(sizes)])

    def ag(b):
        out = [None] * world
        dist.all_gather_object(out, b)
        return out

    for mode, theta in [(m, t) for m in ("pull", "push", "rspush") for t in (64 << 20, 1 << 20, 0)]:
        sync = GradSync(sizes, rank=rank, world=world, device=rank, theta=theta, allgather=ag, dense_mode=mode)
        for it in range(3):
            grads = [o.gen_grads(1000 * it + 17 * r + theta % 97, sizes) for r in range(world)]
            g = torch.from_numpy(grads[rank]).cuda()
            out = torch.empty_like(g)
            gp = [g[int(bounds[i]):int(bounds[i + 1])].data_ptr() for i in range(len(sizes))]
            op = [out[int(bounds[i]):int(bounds[i + 1])].data_ptr() for i in range(len(sizes))]
            sync.dense_step(gp, op)
            torch.cuda.synchronize()
            sync.status()
            ws, wl = o.dense_windows(sizes, 2, theta)
            pools = o.ring_allreduce([o.pack(x, sizes) for x in grads], dtype=F16, windows=(ws, wl))
            got_pool = np.empty_like(pools[rank])  # every rank's pool holds the sums
            cudart.memcpy(got_pool.ctypes.data, sync.last_pool_ptr, got_pool.nbytes)
            cudart.sync_device()
            assert (got_pool == pools[rank]).all(), (mode, theta, it)
            want_pool = o.unpack(pools[rank], world)
            got = out.cpu().numpy()
            for i, s in enumerate(sizes):
                w = want_pool[int(off[i]):int(off[i]) + s]
                assert (got[int(bounds[i]):int(bounds[i + 1])].view(np.uint32) == w.view(np.uint32)).all(), \
                    (mode, theta, it, i)
        sync.close()
    dist.barrier()


@pytest.mark.multigpu(2)
def test_p2p_engine_dense_modes_bit_exact():
    _spawn(_worker_fused, _world())


def _worker_engine_csc(rank, world, port):
    """GradSync.csc_step — the bench's engine path, with the update running beside the
    selection on a second stream — over the reference's own multi-step CSC runs
    (tests/golden/csc_run.npz cases with this world size): hg, the exchanged pool, the next
    important set, hu and w after every iteration, bit for bit."""
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch
    import torch.distributed as dist
    from paper_1902_06855_b200 import cudart
    from paper_1902_06855_b200.engine import GradSync
    torch.cuda.set_device(rank)
    cudart.set_device(rank)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)

    def ag(b):
        out = [None] * world
        dist.all_gather_object(out, b)
        return out

    g = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "csc_run.npz"))
    ran = 0
    for ci, mode in [(c, m) for c in range(int(g["csc_cases"][0])) for m in ("pull", "push")]:
        p = f"c{ci}_"
        n, dt, theta, chunk, T = (int(x) for x in g[p + "meta"])
        if n != world:
            continue
        ran += 1
        sizes = [int(x) for x in g[p + "sizes"]]
        total = sum(sizes)
        sync = GradSync(sizes, rank=rank, world=world, device=rank, dtype=dt, theta=theta, chunk=chunk,
                        csc=True, final_sparsity=0.75, warmup_iters=2, momentum=0.9, lr=0.01,
                        allgather=ag, csc_mode=mode)
        dev = torch.device("cuda", rank)

        def st(name, d):
            ptr, nb = sync.state(name)
            out = np.empty(nb // np.dtype(d).itemsize, d)
            cudart.memcpy(out.ctypes.data, ptr, out.nbytes)
            cudart.sync_device()
            return out

        w0 = np.ascontiguousarray(g[p + "w0"])
        cudart.memcpy(sync.state("w")[0], w0.ctypes.data, w0.nbytes)
        cudart.sync_device()
        bounds = np.concatenate([[0], np.cumsum(sizes)])
        esz = 2 if dt == F16 else 4
        for t in range(T):
            x = torch.from_numpy(np.ascontiguousarray(g[p + "grads"][t][rank])).to(dev)
            sync.csc_step([x[int(bounds[i]):int(bounds[i + 1])].data_ptr() for i in range(len(sizes))])
            torch.cuda.synchronize()
            sync.status()
            want_pool = np.ascontiguousarray(g[p + "pool_x"][t][rank])
            assert (st("pool", np.uint8) == want_pool.view(np.uint8)).all(), (ci, mode, t)
            assert (st("hg", np.uint32) == g[p + "hg"][t][rank].view(np.uint32)).all(), (ci, t)
            assert (st("imp_next", np.uint8) == g[p + "next_imp"][t][rank]).all(), (ci, t)
            assert (st("hu", np.uint32) == g[p + "hu"][t][rank].view(np.uint32)).all(), (ci, t)
            assert (st("w", np.uint32) == g[p + "w"][t][rank].view(np.uint32)).all(), (ci, t)
        sync.close()
    assert ran > 0 or world not in (2, 4)
    dist.barrier()


@pytest.mark.multigpu(2)
def test_p2p_engine_csc_vs_reference_golden():
    _spawn(_worker_engine_csc, _world())


def _worker_overlap(rank, world, port):
    """GradSync.begin_iteration / tensor_complete / finalize_iteration: theta windows
    launched on a communication stream while 'backward' runs, one ring per window; g_avg
    bit-exact against the oracle's windowed ring."""
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch
    import torch.distributed as dist
    from oracle.oracle import RESNET50, Oracle
    from paper_1902_06855_b200 import cudart
    from paper_1902_06855_b200.engine import GradSync
    torch.cuda.set_device(rank)
    cudart.set_device(rank)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)

    def ag(b):
        out = [None] * world
        dist.all_gather_object(out, b)
        return out

    o = Oracle()
    sizes = RESNET50
    off, _, _ = o.pool_layout(sizes, 32000)
    bounds = np.concatenate([[0], np.cumsum(sizes)])
    stream = torch.cuda.current_stream().cuda_stream
    for theta in (8 << 20, 1 << 20):
        sync = GradSync(sizes, rank=rank, world=world, device=rank, theta=theta, allgather=ag)
        for it in range(2):
            grads = [o.gen_grads(300 * it + 7 * r + 5, sizes) for r in range(world)]
            g = torch.from_numpy(grads[rank]).cuda()
            out = torch.empty_like(g)
            gp = [g[int(bounds[i]):int(bounds[i + 1])].data_ptr() for i in range(len(sizes))]
            op = [out[int(bounds[i]):int(bounds[i + 1])].data_ptr() for i in range(len(sizes))]
            sync.begin_iteration(gp, op, stream=stream)
            for tid in range(len(sizes), 0, -1):
                torch.cuda._sleep(2000)  # backward work on the caller's stream
                sync.tensor_complete(tid)
            sync.finalize_iteration()
            torch.cuda.synchronize()
            sync.status()
            ws, wl = o.dense_windows(sizes, 2, theta)
            assert len(ws) > 2
            pools = o.ring_allreduce([o.pack(x, sizes) for x in grads], dtype=F16, windows=(ws, wl))
            want = o.unpack(pools[rank], world)
            got = out.cpu().numpy()
            for i, s in enumerate(sizes):
                assert (got[int(bounds[i]):int(bounds[i + 1])].view(np.uint32) ==
                        want[int(off[i]):int(off[i]) + s].view(np.uint32)).all(), (theta, it, i)
        sync.close()
    dist.barrier()


@pytest.mark.multigpu(2)
def test_p2p_overlapped_windows_bit_exact():
    _spawn(_worker_overlap, _world())


def _worker_tcp_cpp_api(rank, world, port):
    """The reference's C++ API across PROCESSES: TcpTransport (GFL1 over TCP) as the control
    plane, Communicator -> DeviceContext in IPC mode (one GPU per process), ring_allreduce /
    broadcast / FusionEngine over NVLink peer memory — bit-exact vs the oracle, payload
    accounting as the reference's ring (2(N-1) segment_of transfers)."""
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import paper_1902_06855_b200.gflowpy as g
    from oracle.oracle import Oracle
    o = Oracle()
    g.set_device(rank)
    t = g.make_tcp_transport(rank, world, g.tcp_loopback_addresses(world, port))
    comm = g.Communicator(t)
    assert comm.device_mode() == "ipc-p2p", comm.device_mode()
    assert comm.device() == rank
    for it, (L, dt) in enumerate([(1, 1), (97, 1), (1 << 20, 1), (4099, 0), (300_001, 0)]):
        vals = []
        for r in range(world):
            x = np.random.default_rng(500 + 10 * it + r).uniform(-8, 8, L).astype(np.float32)
            vals.append(o.f2h(x) if dt == 1 else x)
        buf = vals[rank].copy()
        before = t.stats().get("ring", {}).get("payload_bytes_sent", 0)
        g.ring_allreduce(comm, buf)
        want = o.ring_allreduce([v.copy() for v in vals], dtype=dt)
        assert (_bits(buf) == _bits(want[rank])).all(), (L, dt)
        sent = t.stats()["ring"]["payload_bytes_sent"] - before
        esz = 2 if dt == 1 else 4
        base, rem = divmod(L, world)
        segs = [base + (1 if j < rem else 0) for j in range(world)]
        p = comm.ring_order.index(rank)
        # RS sends segments p-s, AG sends p+1-s (collectives.cpp:69-96)
        want_sent = sum(segs[(p - s) % world] for s in range(world - 1)) + \
            sum(segs[(p + 1 - s) % world] for s in range(world - 1))
        assert sent == want_sent * esz, (L, sent, want_sent * esz)
    root = world - 1
    b = np.random.default_rng(rank).uniform(-1, 1, 12345).astype(np.float32)
    want_b = np.random.default_rng(root).uniform(-1, 1, 12345).astype(np.float32)
    g.broadcast(comm, b, root)
    assert (b.view(np.uint32) == want_b.view(np.uint32)).all()
    t.barrier()


@pytest.mark.multigpu(2)
def test_tcp_transport_cpp_api_across_processes():
    _spawn(_worker_tcp_cpp_api, _world())

# SPDX-License-Identifier: Apache-2.0
"""Stress of the cross-rank ordering: thousands of back-to-back steps, no host sync between them.

Every step picks (the same on every rank, from a shared seed) one engine — dense rspush
(theta 0 / 64 KiB / inf), dense pull, dense push-pull ring, CSC push form, CSC pull form — and one
of eight gradient sets carrying NaN / inf / fp16-overflow values, while bf16 GEMMs run on another
stream of the same GPU. The step's results are copied (async, device-to-device) into a history
ring; every batch the host synchronises once and checks each recorded step bit for bit against the
CPU oracle: the pool and g_avg (dense), the exchanged pool and the next selected set (CSC, oracle
run in lockstep). This exercises the fence-free publication of the routed pack's NVLink stores
(push.cu), the epoch/flag protocol under reuse, pool alternation (pull) and the inbox reuse
ordering (rspush, select) — see DESIGN.md §6 for the ordering argument this backs.

  * test_stress_colocated   N = 2 and 4 ranks on ONE B200 (gf_comm_connect_colocated).
  * test_stress_multigpu    one process per GPU over NVLink (N = the box's GPUs, up to 4).
"""
import ctypes as C
import os
import socket

import numpy as np
import pytest

pytestmark = [pytest.mark.gpu]

F16 = 1
THETA_INF = (1 << 64) - 1
SIZES = [5, 97, 1, 4099, 30_001, 8, 77, 3, 65536, 1000, 120_000, 7, 257, 50_000, 2048, 99_999]
CHUNK = 1000
ENGINES = [  # (kind, mode, theta)
    ("dense", "rspush", THETA_INF), ("dense", "rspush", 64 << 10), ("dense", "rspush", 0),
    ("dense", "pull", THETA_INF), ("dense", "push", 1 << 17),
    ("csc", "push", THETA_INF), ("csc", "pull", 20_000),
]
NSETS = 8


def make_sets(o, world, nan=True):
    """NSETS gradient sets per rank with special values (seeded: identical in every process).
    CSC takes nan=False: a NaN chunk norm leaves the reference's partial_sort order unspecified
    (DESIGN.md §2), so its selection has no single right answer to check against."""
    sets = []
    for s in range(NSETS):
        per = []
        for r in range(world):
            g = o.gen_grads(7000 + 97 * s + r, SIZES) * np.float32(1 + s % 3)
            rng = np.random.default_rng(11 * s + r)
            idx = rng.integers(0, g.size, 64)
            if nan:
                g[idx[:16]] = np.nan
            g[idx[16:24]] = np.inf
            g[idx[24:32]] = -np.inf
            g[idx[32:]] *= np.float32(4e4)  # fp16 overflow -> clamped sums
            per.append(g)
        sets.append(per)
    return sets


class Expect:
    """Oracle results: dense (engine theta, set) -> per-rank pool / flat g_avg; CSC lockstep state."""

    def __init__(self, o, world, sets, csc_sets, ranks):
        self.o, self.world, self.sets, self.csc_sets, self.ranks = o, world, sets, csc_sets, ranks
        self.off, self.nc, _ = o.pool_layout(SIZES, CHUNK)
        self.total = int(sum(SIZES))
        self.dense = {}
        self.csc = {}

    def dense_result(self, theta, s):
        key = (theta, s)
        if key not in self.dense:
            o = self.o
            ws, wl = o.dense_windows(SIZES, 2, theta)
            pools = o.ring_allreduce([o.pack(g, SIZES, dtype=F16) for g in self.sets[s]], dtype=F16, windows=(ws, wl))
            out = {}
            for r in self.ranks:
                gavg = o.unpack(pools[r], self.world, dtype=F16)
                flat = np.concatenate([gavg[int(a):int(a) + n] for a, n in zip(self.off, SIZES)])
                out[r] = (pools[r], flat)
            self.dense[key] = out
        return self.dense[key]

    def csc_step(self, eidx, theta, s):
        """Advance engine eidx's oracle state by one CSC iteration on set s; returns per-rank
        (exchanged pool, next important set)."""
        o = self.o
        st = self.csc.setdefault(eidx, dict(t=0, imp=np.ones(self.nc, np.uint8),
                                             hg=[np.zeros(self.total, np.float32) for _ in range(self.world)]))
        t = st["t"]
        k = o.selection_count(o.sparsity_at(t + 1, 3, 0.75), self.nc)
        pools, _, nxt, _ = o.csc_iteration(self.csc_sets[s], SIZES, CHUNK, theta, np.float32(0.9), st["imp"], k, st["hg"],
                                           dtype=F16)
        st["imp"] = nxt
        st["t"] = t + 1
        return {r: (pools[r], nxt) for r in self.ranks}


def run_stress(engines_by_rank, streams, ranks, world, steps, batch, seed, barrier, load_stream=None):
    """engines_by_rank[r][e]: rank r's GradSync for ENGINES[e] (r in ranks). One host thread."""
    import torch
    from oracle.oracle import Oracle
    from paper_1902_06855_b200 import cudart
    o = Oracle()
    sets = make_sets(o, world)
    csc_sets = make_sets(o, world, nan=False)
    exp = Expect(o, world, sets, csc_sets, ranks)
    total, nc = exp.total, exp.nc
    bounds = np.concatenate([[0], np.cumsum(SIZES)])
    dev = {r: [torch.from_numpy(x[s][r]).cuda() for x in (sets, csc_sets) for s in range(NSETS)] for r in ranks}

    def table(flat):
        return (C.c_void_p * len(SIZES))(*[flat[int(bounds[i]):int(bounds[i + 1])].data_ptr() for i in range(len(SIZES))])

    gtab = {r: [table(x) for x in dev[r]] for r in ranks}
    outs = {r: torch.empty(total, device="cuda") for r in ranks}
    otab = {r: table(outs[r]) for r in ranks}
    # history ring: pool (u16) + g_avg / selected set per recorded step
    hist_pool = {r: torch.empty((batch, total), dtype=torch.int16, device="cuda") for r in ranks}
    hist_out = {r: torch.empty((batch, total), dtype=torch.float32, device="cuda") for r in ranks}
    hist_imp = {r: torch.empty((batch, nc), dtype=torch.uint8, device="cuda") for r in ranks}
    A = torch.randn(2048, 2048, dtype=torch.bfloat16, device="cuda")
    Bm = torch.randn(2048, 2048, dtype=torch.bfloat16, device="cuda")
    rng = np.random.default_rng(seed)
    torch.cuda.synchronize()
    checked = 0
    for b0 in range(0, steps, batch):
        plan = [(int(rng.integers(0, len(ENGINES))), int(rng.integers(0, NSETS))) for _ in range(min(batch, steps - b0))]
        if load_stream is not None:  # concurrent GEMM load on the same GPU
            with torch.cuda.stream(load_stream):
                for _ in range(8):
                    torch.matmul(A, Bm)
        for i, (e, s) in enumerate(plan):
            kind = ENGINES[e][0]
            for r in ranks:
                g = engines_by_rank[r][e]
                st = streams[r]
                if kind == "dense":
                    g.dense_step(gtab[r][s], otab[r], stream=st)  # sets 0..NSETS-1: with NaNs
                    cudart.memcpy(hist_out[r][i].data_ptr(), outs[r].data_ptr(), total * 4, st)
                else:
                    g.csc_step(gtab[r][NSETS + s], stream=st)  # the NaN-free copies
                    p, n = g.state("imp_next")
                    cudart.memcpy(hist_imp[r][i].data_ptr(), p, nc, st)
                p, n = g.state("pool")
                cudart.memcpy(hist_pool[r][i].data_ptr(), p, total * 2, st)
        for r in ranks:
            cudart.stream_sync(streams[r])
            for g in engines_by_rank[r]:
                g.status()
        hp = {r: hist_pool[r].cpu().numpy().view(np.uint16) for r in ranks}
        ho = {r: hist_out[r].cpu().numpy() for r in ranks}
        hi = {r: hist_imp[r].cpu().numpy() for r in ranks}
        for i, (e, s) in enumerate(plan):
            kind, mode, theta = ENGINES[e]
            if kind == "dense":
                want = exp.dense_result(theta, s)
                for r in ranks:
                    assert (hp[r][i] == want[r][0]).all(), ("pool", b0 + i, ENGINES[e], s, r)
                    assert (ho[r][i].view(np.uint32) == want[r][1].view(np.uint32)).all(), ("g_avg", b0 + i, e, s, r)
            else:
                want = exp.csc_step(e, theta, s)
                for r in ranks:
                    assert (hp[r][i] == want[r][0]).all(), ("csc pool", b0 + i, ENGINES[e], s, r)
                    assert (hi[r][i] == want[r][1]).all(), ("csc set", b0 + i, ENGINES[e], s, r)
            checked += 1
        barrier()
    return checked


def build_engines(GradSync, make):
    return [make(kind, mode, theta) for kind, mode, theta in ENGINES]


@pytest.mark.parametrize("world,steps", [(2, 1500), (4, 600)])
def test_stress_colocated(world, steps):
    import torch
    from colo import ColoWorld  # noqa: F401  (conftest env: eager loading, 32 connections)
    from paper_1902_06855_b200 import cudart
    from paper_1902_06855_b200.engine import GradSync
    per_engine = []
    for kind, mode, theta in ENGINES:
        kw = dict(theta=theta, chunk=CHUNK, timeout_ms=20000)
        if kind == "dense":
            kw["dense_mode"] = mode
        else:
            kw.update(csc=True, csc_mode=mode, final_sparsity=0.75, warmup_iters=3)
        per_engine.append(GradSync.colocated(world, SIZES, device=torch.cuda.current_device(), **kw))
    engines_by_rank = {r: [per_engine[e][r] for e in range(len(ENGINES))] for r in range(world)}
    streams = {r: cudart.stream_create() for r in range(world)}
    load = torch.cuda.Stream()
    try:
        n = run_stress(engines_by_rank, streams, list(range(world)), world, steps, 50, 1234 + world,
                       lambda: None, load_stream=load)
        assert n == steps
    finally:
        for g in [g for ranks in per_engine for g in ranks]:
            g.close()
        for s in streams.values():
            cudart.stream_sync(s)
            cudart.stream_destroy(s)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, steps):
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

    engines = []
    for kind, mode, theta in ENGINES:
        kw = dict(theta=theta, chunk=CHUNK, timeout_ms=20000, rank=rank, world=world, device=rank, allgather=ag)
        if kind == "dense":
            kw["dense_mode"] = mode
        else:
            kw.update(csc=True, csc_mode=mode, final_sparsity=0.75, warmup_iters=3)
        engines.append(GradSync(SIZES, **kw))
    stream = cudart.stream_create()
    n = run_stress({rank: engines}, {rank: stream}, [rank], world, steps, 100, 4321 + world, dist.barrier,
                   load_stream=torch.cuda.Stream())
    assert n == steps
    for g in engines:
        g.close()
    dist.barrier()


@pytest.mark.multigpu(2)
def test_stress_multigpu():
    import torch
    import torch.multiprocessing as mp
    world = min(torch.cuda.device_count(), 4)
    mp.spawn(_worker, args=(world, _free_port(), 5000), nprocs=world, join=True)

# SPDX-License-Identifier: Apache-2.0
"""CPU, world_size 2 over gloo: the host-side logic of the multi-GPU path.

Every rank must derive the SAME collective geometry independently (pool layout, theta
windows, segment_of splits, CSC selection counts): the NVLink kernels pair CTA b with CTA b
and owner j with segment j without exchanging any of it. Also runs bench.py's reference arm
under a 2-rank torchrun-style launch (rank 0 times the reference CPU path, rank 1 exits 0).
"""
import json
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    from paper_1902_06855_b200.engine import (PoolLayout, dense_windows, selection_count,
                                              sparsity_at)
    import bench
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    geo = {}
    for name, sizes in (("alexnet", bench.ALEXNET), ("resnet50", bench.RESNET50)):
        L = PoolLayout.build(sizes, 32000)
        for theta in (0, 1 << 20, 64 << 20, bench.THETA_INF):
            ws, wl = dense_windows(L, 2, theta)
            segs = [[(wl_ // world) * j + min(j, wl_ % world) for j in range(world)] for wl_ in wl]
            geo[f"{name}/{theta}"] = (L.num_chunks, ws, wl, segs)
        geo[f"{name}/k"] = [selection_count(sparsity_at(t, 3, 0.9), L.num_chunks) for t in range(6)]
    out = [None] * world
    dist.all_gather_object(out, geo)
    q.put((rank, all(o == out[0] for o in out), out[0]["alexnet/k"], out[0]["resnet50/k"]))
    dist.destroy_process_group()


def test_geometry_identical_on_every_rank():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = [q.get(timeout=120) for _ in ps]
    for p in ps:
        p.join(60)
        assert p.exitcode == 0
    assert all(ok for _, ok, _, _ in res)
    _, _, k_alex, k_res = res[0]
    assert k_alex[0] == 1909 and k_alex[-1] == 191  # iteration 0 dense ramp -> 10 % of 1909
    assert k_res[-1] == 80


def test_engine_layout_matches_oracle(oracle):
    from paper_1902_06855_b200.engine import PoolLayout, dense_windows
    import bench
    for sizes in (bench.ALEXNET, bench.RESNET50, [10], [70000], [3, 2, 1]):
        L = PoolLayout.build(sizes, 32000 if len(sizes) > 3 else 4)
        off, nc, _ = oracle.pool_layout(sizes, L.chunk)
        assert list(L.offsets) == [int(x) for x in off] and L.num_chunks == nc
        for theta in (0, 96, 4096, 1 << 20, bench.THETA_INF):
            ws, wl = dense_windows(L, 2, theta)
            ows, owl = oracle.dense_windows(sizes, 2, theta)
            assert ws == [int(x) for x in ows] and wl == [int(x) for x in owl]


@pytest.mark.skipif(not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libgflowref.so")),
                    reason="oracle/_ref not built")
def test_bench_reference_arm_two_ranks():
    """`torchrun --nproc-per-node 2 bench.py --impl reference`: one JSON line from rank 0."""
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_port()), WORLD_SIZE="2")
    outs = []
    procs = []
    for r in range(2):
        e = dict(env, RANK=str(r), LOCAL_RANK=str(r))
        procs.append(subprocess.Popen([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                                       "--gpus", "2", "--steps", "1", "--warmup", "1",
                                       "--workload", "resnet50-dense"],
                                      cwd=ROOT, env=e, stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True))
    for p in procs:
        o, err = p.communicate(timeout=600)
        assert p.returncode == 0, err[-2000:]
        outs.append(o)
    lines = [json.loads(x) for x in outs[0].splitlines() if x.startswith("{")]
    assert len(lines) == 1 and not outs[1].strip()
    d = lines[0]
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["unit"] == "ms" and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "reference" and d["e2e"]["h2d_bytes_per_step"] == 0


def test_bench_numa_bind_is_best_effort():
    """bench.numa_bind never raises: without a GPU (or sysfs/affinity rights) it returns None and
    leaves the process affinity alone."""
    import torch
    import bench
    before = os.sched_getaffinity(0)
    out = bench.numa_bind(torch, 0)
    assert out is None or (set(out) == {"gpu_pci", "numa_node", "cpus"} and out["cpus"] >= 1)
    if out is None:
        assert os.sched_getaffinity(0) == before

# SPDX-License-Identifier: Apache-2.0
"""Generate the golden fixtures in tests/golden/ from the UNMODIFIED reference.

Run in the build container (needs oracle/_ref/libgflowref.so, i.e. /root/reference):

    make -C oracle && python tests/golden/gen_golden.py

Every array here comes out of the reference library's own public C++ API driven by
oracle/ref_driver.cpp (ranks as threads over its InprocTransport). Inputs are
seeded numpy draws stored alongside the outputs, so the fixtures are
self-contained and travel to the GPU box with the repo.
"""
from __future__ import annotations

import concurrent.futures as cf
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle.oracle import ALEXNET, RESNET50, THETA_INF, Reference  # noqa: E402


def specials(rng, n, nan=True):
    """fp32 values that exercise the codec's corner cases (half.hpp:20-59). CSC fixtures
    use nan=False: a NaN chunk norm makes the reference's partial_sort order unspecified."""
    base = rng.uniform(-1, 1, n).astype(np.float32)
    pick = rng.integers(0 if nan else 2, 12, n)
    table = np.array([np.nan, -np.nan, np.inf, -np.inf, 70000.0, -70000.0, 65504.0, 65520.0,
                      2.0 ** -25, 3e-8, -0.0, 1.0 + 2.0 ** -11], np.float32)
    mask = rng.random(n) < 0.02
    base[mask] = table[pick[mask]]
    return base


def codec(ref: Reference, out):
    # exhaustive digest of float_to_half_bits over all 2^32 fp32 patterns, in 64 slices
    slices = 64
    per = (1 << 32) // slices
    with cf.ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        parts = list(ex.map(lambda i: ref.codec_digest(i * per, per), range(slices)))
    out["codec_digest_slices"] = np.array(parts, np.uint64)
    out["codec_digest_all"] = np.array([sum(parts) % (1 << 64)], np.uint64)
    h = np.arange(65536, dtype=np.uint16)
    out["decode_table_bits"] = ref.h2f(h).view(np.uint32)
    kat_in = np.array([0.0, -0.0, 1.0, 70000.0, -70000.0, np.inf, -np.inf, np.nan,
                       1.0 + 2.0 ** -11, 1.0 + 3 * 2.0 ** -11, 2.0 ** -24, 65504.0, 65519.0,
                       65520.0, 2.0 ** -25, 1.5 * 2.0 ** -25, 6.1e-5, -3.0e-6], np.float32)
    out["kat_in"] = kat_in
    out["kat_out"] = ref.f2h(kat_in)
    rng = np.random.default_rng(11)
    x = specials(rng, 4096)
    out["acc_a"] = ref.f2h(x)
    out["acc_b"] = ref.f2h(specials(rng, 4096) * 3e4)
    d = out["acc_a"].copy()
    ref.accumulate(d, out["acc_b"], dtype=1)
    out["acc_out"] = d
    fa = rng.standard_normal(4096).astype(np.float32)
    fb = rng.standard_normal(4096).astype(np.float32)
    fa[::97] = np.inf
    fb[::97] = -np.inf
    fb[5::101] = np.nan
    out["acc32_a"], out["acc32_b"] = fa, fb
    d32 = fa.copy()
    ref.accumulate(d32, fb, dtype=0)
    out["acc32_out"] = d32


def layouts(ref: Reference, out):
    for name, sizes in [("alexnet", ALEXNET), ("resnet50", RESNET50)]:
        off, nc, lens = ref.pool_layout(sizes, 32000)
        out[f"{name}_sizes"] = np.array(sizes, np.uint64)
        out[f"{name}_offsets"] = off
        out[f"{name}_nc"] = np.array([nc], np.uint64)
        out[f"{name}_chunk_lens"] = lens
    cases = [(0.0, 10), (0.5, 4), (0.99, 10), (0.85, 1903), (0.9, 1903), (0.9, 1909), (0.9, 799),
             (0.85, 1909), (0.85, 799), (0.75, 6), (0.5, 5), (0.5, 3), (0.25, 2), (0.995, 100)]
    out["selcount_s"] = np.array([c[0] for c in cases])
    out["selcount_nc"] = np.array([c[1] for c in cases], np.uint64)
    out["selcount_k"] = np.array([ref.L.refd_selection_count(c[0], c[1]) for c in cases], np.uint64)


def dense(ref: Reference, out):
    rng = np.random.default_rng(5)
    cases = []
    for n in (2, 3, 4, 8):
        for dt in (1, 0):
            for theta in (0, 96, 4096, THETA_INF):
                cases.append(([13, 29, 7, 41, 11], n, dt, theta))
    big = [1000, 64, 3000, 5, 8192]
    cases += [(big, 2, 1, 4096), (big, 3, 0, THETA_INF), (big, 8, 1, 0), (big, 4, 1, THETA_INF)]
    for ci, (sizes, n, dt, theta) in enumerate(cases):
        grads = [specials(rng, sum(sizes)) * np.float32(rng.uniform(0.5, 20)) for _ in range(n)]
        pools, gavg, wb, sent = ref.dense_sync(grads, sizes, dtype=dt, theta=theta)
        p = f"d{ci}_"
        out[p + "meta"] = np.array([n, dt, theta], np.uint64)
        out[p + "sizes"] = np.array(sizes, np.uint64)
        out[p + "grads"] = np.stack(grads)
        out[p + "pools"] = np.stack(pools)
        out[p + "gavg"] = np.stack(gavg)
        out[p + "window_bytes"] = wb
        out[p + "sent"] = sent
    out["dense_cases"] = np.array([len(cases)])


def csc(ref: Reference, out):
    rng = np.random.default_rng(7)
    cases = [([300, 50, 1000, 7], 100, 2, 1, THETA_INF), ([300, 50, 1000, 7], 100, 3, 1, 400),
             ([64] * 20, 16, 4, 1, 0), ([5000, 3], 1000, 2, 0, THETA_INF),
             ([4000, 96, 2000], 512, 8, 1, 2048)]
    for ci, (sizes, chunk, n, dt, theta) in enumerate(cases):
        T = 4
        steps = [[specials(rng, sum(sizes), nan=False) * np.float32(rng.uniform(0.1, 3)) for _ in range(n)]
                 for _ in range(T)]
        w0 = rng.uniform(-1, 1, sum(sizes)).astype(np.float32)
        res = ref.csc_run(steps, sizes, chunk, dtype=dt, theta=theta, final_sparsity=0.75,
                          warmup=2, momentum=0.9, lr=0.01, weights0=w0)
        p = f"c{ci}_"
        out[p + "meta"] = np.array([n, dt, theta, chunk, T], np.uint64)
        out[p + "sizes"] = np.array(sizes, np.uint64)
        out[p + "grads"] = np.array(steps)            # [T, n, total]
        out[p + "w0"] = w0
        for k in ("pool_corr", "hg", "pool_x", "norms_loc", "norms_sum", "imp", "next_imp", "hu", "w"):
            out[p + k] = np.array(res[k])              # [T, n, ...]
        out[p + "checksum"] = res["checksum"]
        out[p + "windows"] = res["windows"]
    out["csc_cases"] = np.array([len(cases)])


def hand_traces(ref: Reference, out):
    """test_sparse.cpp:198-233 — bit-set {0,3} and ties -> {0,1} (fp32 pools, chunk 1)."""
    r = ref.csc_run([[np.array([1, 0, 2, 0], np.float32), np.array([1, 0, 0, 4], np.float32)]],
                    [4], 1, dtype=0, final_sparsity=0.5, momentum=0.0)
    out["trace_bitset"] = r["next_imp"][0][0]
    r = ref.csc_run([[np.array([3, 3, 3, 3], np.float32)]], [4], 1, dtype=0, final_sparsity=0.5,
                    momentum=0.0)
    out["trace_ties"] = r["next_imp"][0][0]


TRAIN_CASES = [
    dict(ranks=2, model_dims=[8, 1], task="logistic", iterations=40, n_examples=128, batch=16,
         learning_rate=0.3, seed=7),
    dict(ranks=4, iterations=12, chunk_size=100),
    dict(ranks=4, iterations=12, chunk_size=100, csc=True, final_sparsity=0.85, warmup_iters=3),
    dict(ranks=2, iterations=10, precision="fp16", theta_bytes=2048),
    dict(ranks=3, model_dims=[16, 24, 8, 1], iterations=8, precision="fp16", csc=True,
         final_sparsity=0.75, warmup_iters=2, chunk_size=64, n_examples=96, batch=8),
    dict(ranks=4, model_dims=[32, 16, 1], iterations=6, theta_bytes=0),
]


def train_runs(ref: Reference, out):
    """Whole training runs of the reference trainer (train_worker), rank 0's view."""
    for i, c in enumerate(TRAIN_CASES):
        r = ref.train(**c)
        out[f"t{i}_loss"] = r["loss"]
        out[f"t{i}_grad_bytes"] = r["grad_payload_bytes"]
        out[f"t{i}_weights"] = r["final_weights"]
    out["train_cases"] = np.array([len(TRAIN_CASES)])
    out["cases_json"] = np.array(json.dumps(TRAIN_CASES))


REDUCE_CASES = [  # (n, dtype, len, root, ring_order or None)
    (2, 0, 37, 0, None), (2, 1, 1000, 1, None), (3, 0, 1001, 2, None), (4, 1, 4099, 1, [2, 0, 3, 1]),
    (5, 1, 3, 4, None), (8, 0, 777, 5, [7, 6, 5, 4, 3, 2, 1, 0]), (8, 1, 8192, 0, None),
]
HIER_CASES = [  # (n, group_size, dtype, len)
    (4, 2, 0, 1000), (4, 2, 1, 4099), (6, 3, 1, 777), (6, 2, 0, 9), (8, 2, 0, 16384), (8, 4, 1, 5000),
    (4, 1, 1, 100), (4, 4, 0, 100),
]


def rooted(ref: Reference, out):
    """reduce() end states of every rank and hierarchical_allreduce results + payloads."""
    rng = np.random.default_rng(21)

    def inputs(n, dt, length):
        xs = [specials(rng, length) * np.float32(4.0) for _ in range(n)]
        return [ref.f2h(x) if dt == 1 else x for x in xs]

    for i, (n, dt, length, root, ring) in enumerate(REDUCE_CASES):
        bufs = inputs(n, dt, length)
        out[f"r{i}_in"] = np.stack(bufs)
        work = [b.copy() for b in bufs]
        out[f"r{i}_sent"] = ref.reduce(work, root, dtype=dt, ring_order=ring)
        out[f"r{i}_out"] = np.stack(work)
    for i, (n, m, dt, length) in enumerate(HIER_CASES):
        bufs = inputs(n, dt, length)
        out[f"h{i}_in"] = np.stack(bufs)
        work = [b.copy() for b in bufs]
        out[f"h{i}_sent"] = ref.allreduce(work, dtype=dt, algo=1, group_size=m)
        out[f"h{i}_out"] = np.stack(work)
    out["cases_json"] = np.array(json.dumps({"reduce": REDUCE_CASES, "hier": HIER_CASES}))


def main():
    ref = Reference()
    only = set(sys.argv[1:])
    if only:  # e.g. `gen_golden.py rooted`: regenerate just those fixtures
        if "rooted" in only:
            r: dict = {}
            rooted(ref, r)
            np.savez_compressed(os.path.join(HERE, "rooted.npz"), **r)
            print("rooted.npz", os.path.getsize(os.path.join(HERE, "rooted.npz")))
        return
    out: dict = {}
    codec(ref, out)
    layouts(ref, out)
    hand_traces(ref, out)
    np.savez_compressed(os.path.join(HERE, "codec_layout.npz"), **out)
    d: dict = {}
    dense(ref, d)
    np.savez_compressed(os.path.join(HERE, "dense_sync.npz"), **d)
    c: dict = {}
    csc(ref, c)
    np.savez_compressed(os.path.join(HERE, "csc_run.npz"), **c)
    t: dict = {}
    train_runs(ref, t)
    np.savez_compressed(os.path.join(HERE, "train.npz"), **t)
    r: dict = {}
    rooted(ref, r)
    np.savez_compressed(os.path.join(HERE, "rooted.npz"), **r)
    for f in ("codec_layout.npz", "dense_sync.npz", "csc_run.npz", "train.npz", "rooted.npz"):
        print(f, os.path.getsize(os.path.join(HERE, f)))


if __name__ == "__main__":
    main()

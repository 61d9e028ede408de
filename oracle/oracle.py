# SPDX-License-Identifier: Apache-2.0
"""CPU ORACLE loader — TEST INFRASTRUCTURE ONLY.

numpy/ctypes front end for
  * ``liboracle.so``  — the C restatement in gf_oracle.c (always built), and
  * ``_ref/libgflowref.so`` — the UNMODIFIED reference library plus our C shim
    (ref_driver.cpp), present when oracle/Makefile could see /root/reference
    (the built .so travels to the GPU box).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this module, and only as the checker or
the timed CPU baseline. The product package never imports it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
THETA_INF = (1 << 64) - 1

_u64p = C.POINTER(C.c_uint64)
_f32p = C.POINTER(C.c_float)
_u8p = C.POINTER(C.c_uint8)
_vp = C.c_void_p


def build(quiet: bool = True) -> None:
    """make -C oracle (restatement always; reference when /root/reference exists)."""
    out = subprocess.run(["make", "-C", HERE, "-j8"], capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("oracle build failed:\n" + out.stdout[-4000:] + out.stderr[-4000:])


def _load(path):
    if not os.path.exists(path):
        return None
    return C.CDLL(path)


def np_ptr(a: np.ndarray):
    return a.ctypes.data_as(_vp)


def ptr_array(arrs):
    return (_vp * len(arrs))(*[None if a is None else a.ctypes.data for a in arrs])


def u64(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.uint64))


class Oracle:
    """The C restatement (gf_oracle.c)."""

    def __init__(self):
        path = os.path.join(HERE, "liboracle.so")
        if not os.path.exists(path):
            build()
        L = C.CDLL(path)
        self.L = L
        L.go_f2h.restype = C.c_uint16
        L.go_f2h.argtypes = [C.c_float]
        L.go_h2f.restype = C.c_float
        L.go_h2f.argtypes = [C.c_uint16]
        L.go_codec_digest.restype = C.c_uint64
        L.go_codec_digest.argtypes = [C.c_uint64, C.c_uint64, C.c_int]
        L.go_pool_layout.restype = C.c_uint64
        L.go_pool_layout.argtypes = [_vp, C.c_int, C.c_uint64, _vp]
        L.go_chunk_l1.restype = C.c_float
        L.go_chunk_l1.argtypes = [C.c_int, _vp, C.c_uint64, C.c_uint64]
        L.go_selection_count.restype = C.c_uint64
        L.go_selection_count.argtypes = [C.c_double, C.c_uint64]
        L.go_sparsity_at.restype = C.c_double
        L.go_sparsity_at.argtypes = [C.c_uint64, C.c_uint64, C.c_double]
        L.go_fnv1a.restype = C.c_uint64
        L.go_fnv1a.argtypes = [_vp, C.c_uint64]
        L.go_dense_windows.restype = C.c_int
        L.go_dense_windows.argtypes = [_vp, C.c_int, C.c_uint64, C.c_uint64, _vp, _vp, C.c_int]
        L.go_csc_windows.restype = C.c_int
        L.go_csc_windows.argtypes = [_vp, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64,
                                     C.c_uint64, _vp, _vp, C.c_int]
        L.go_csc_iteration.restype = C.c_int
        L.go_csc_iteration.argtypes = [C.c_int, C.c_int, _vp, C.c_int, C.c_uint64, C.c_uint64,
                                       C.c_float, _vp, _vp, _vp, _vp, _vp, _vp, C.c_uint64, _vp]
        for name, args in {
            "go_f2h_array": [_vp, _vp, C.c_uint64],
            "go_h2f_array": [_vp, _vp, C.c_uint64],
            "go_accumulate": [C.c_int, _vp, _vp, C.c_uint64],
            "go_pack": [C.c_int, _vp, _vp, C.c_int, _vp, C.c_float],
            "go_unpack": [C.c_int, _vp, C.c_uint64, C.c_int, _vp],
            "go_ring_allreduce": [C.c_int, _vp, C.c_int, C.c_uint64, _vp],
            "go_ring_allreduce_windows": [C.c_int, _vp, C.c_int, _vp, _vp, C.c_int, _vp],
            "go_ring_reduce": [C.c_int, _vp, C.c_int, C.c_int, C.c_uint64],
            "go_hier_allreduce": [C.c_int, _vp, C.c_int, C.c_int, C.c_uint64],
            "go_chunk_norms": [C.c_int, _vp, C.c_uint64, C.c_uint64, C.c_uint64, _vp, C.c_int, _vp],
            "go_csc_correct": [C.c_int, _vp, _vp, _vp, C.c_uint64, C.c_uint64, C.c_uint64, C.c_float],
            "go_csc_scatter": [C.c_int, _vp, _vp, C.c_uint64, C.c_uint64, C.c_uint64, _vp],
            "go_select_topk": [_vp, C.c_uint64, C.c_uint64, _vp],
            "go_csc_sgd_update": [C.c_int, _vp, _vp, C.c_uint64, C.c_uint64, C.c_uint64, C.c_int,
                                  C.c_float, C.c_float, _vp, _vp],
            "go_gen_grads": [C.c_uint64, _vp, C.c_int, _vp],
        }.items():
            f = getattr(L, name)
            f.restype = None
            f.argtypes = args
        L.go_csc_compact.restype = C.c_uint64
        L.go_csc_compact.argtypes = [C.c_int, _vp, _vp, C.c_uint64, C.c_uint64, C.c_uint64, _vp]

    # -- codec ---------------------------------------------------------------
    def f2h(self, x) -> np.ndarray:
        x = np.ascontiguousarray(np.asarray(x, dtype=np.float32))
        out = np.empty(x.shape, np.uint16)
        self.L.go_f2h_array(np_ptr(x), np_ptr(out), x.size)
        return out

    def h2f(self, h) -> np.ndarray:
        h = np.ascontiguousarray(np.asarray(h, dtype=np.uint16))
        out = np.empty(h.shape, np.float32)
        self.L.go_h2f_array(np_ptr(h), np_ptr(out), h.size)
        return out

    def codec_digest(self, first=0, count=1 << 32, nthreads=None) -> int:
        return int(self.L.go_codec_digest(first, count, nthreads or os.cpu_count() or 1))

    # -- layout --------------------------------------------------------------
    def pool_layout(self, sizes, chunk):
        s = u64(sizes)
        off = np.zeros(len(s), np.uint64)
        nc = int(self.L.go_pool_layout(np_ptr(s), len(s), chunk, np_ptr(off)))
        total = int(s.sum())
        lens = np.full(nc, chunk, np.uint64)
        if nc:
            lens[-1] = total - (nc - 1) * chunk
        return off, nc, lens

    def dense_windows(self, sizes, esz, theta):
        s = u64(sizes)
        cap = len(s) + 2
        ws, wl = np.zeros(cap, np.uint64), np.zeros(cap, np.uint64)
        n = self.L.go_dense_windows(np_ptr(s), len(s), esz, theta, np_ptr(ws), np_ptr(wl), cap)
        return ws[:n].copy(), wl[:n].copy()

    def csc_windows(self, imp, total, chunk, esz, theta):
        imp = np.ascontiguousarray(imp, dtype=np.uint8)
        cap = len(imp) + 2
        ws, wl = np.zeros(cap, np.uint64), np.zeros(cap, np.uint64)
        n = self.L.go_csc_windows(np_ptr(imp), total, chunk, len(imp), esz, theta,
                                  np_ptr(ws), np_ptr(wl), cap)
        return ws[:n].copy(), wl[:n].copy()

    # -- path pieces -----------------------------------------------------------
    def pack(self, flat_asc, sizes, dtype=1, scale=1.0):
        g = np.ascontiguousarray(flat_asc, dtype=np.float32)
        s = u64(sizes)
        pool = np.zeros(int(s.sum()), np.uint16 if dtype == 1 else np.float32)
        self.L.go_pack(dtype, np_ptr(g), np_ptr(s), len(s), np_ptr(pool), scale)
        return pool

    def unpack(self, pool, world, dtype=1):
        out = np.empty(pool.size, np.float32)
        self.L.go_unpack(dtype, np_ptr(pool), pool.size, world, np_ptr(out))
        return out

    def ring_allreduce(self, bufs, dtype=1, windows=None, ring_order=None):
        """In place on a list of per-rank numpy buffers."""
        n = len(bufs)
        ro = None if ring_order is None else np.ascontiguousarray(ring_order, dtype=np.int32)
        if windows is None:
            self.L.go_ring_allreduce(dtype, ptr_array(bufs), n, bufs[0].size,
                                     None if ro is None else np_ptr(ro))
        else:
            ws, wl = u64(windows[0]), u64(windows[1])
            self.L.go_ring_allreduce_windows(dtype, ptr_array(bufs), n, np_ptr(ws), np_ptr(wl),
                                             len(ws), None if ro is None else np_ptr(ro))
        return bufs

    def ring_reduce(self, bufs, root, dtype=1, ring_order=None):
        """reduce(comm, buf, root) end state (collectives.cpp:99-144, 229-235), in place on
        per-RANK buffers; ring_order maps ring position -> rank (identity when None)."""
        n = len(bufs)
        ring = list(range(n)) if ring_order is None else [int(x) for x in ring_order]
        by_pos = [bufs[ring[t]] for t in range(n)]
        self.L.go_ring_reduce(dtype, ptr_array(by_pos), n, ring.index(root), bufs[0].size)
        return bufs

    def hier_allreduce(self, bufs, group_size, dtype=1):
        """hierarchical_allreduce (collectives.cpp:179-201), in place on per-rank buffers."""
        self.L.go_hier_allreduce(dtype, ptr_array(bufs), len(bufs), group_size, bufs[0].size)
        return bufs

    def chunk_norms(self, pool, chunk, nc, imp, world, dtype=1):
        out = np.empty(nc, np.float32)
        impa = None if imp is None else np.ascontiguousarray(imp, dtype=np.uint8)
        self.L.go_chunk_norms(dtype, np_ptr(pool), pool.size, chunk, nc,
                              None if impa is None else np_ptr(impa), world, np_ptr(out))
        return out

    def csc_correct(self, pool, hg, imp, chunk, momentum, dtype=1):
        imp = np.ascontiguousarray(imp, dtype=np.uint8)
        self.L.go_csc_correct(dtype, np_ptr(pool), np_ptr(hg), np_ptr(imp), pool.size, chunk,
                              len(imp), momentum)

    def csc_compact(self, pool, imp, chunk, dtype=1):
        imp = np.ascontiguousarray(imp, dtype=np.uint8)
        st = np.zeros(pool.size, pool.dtype)
        n = self.L.go_csc_compact(dtype, np_ptr(pool), np_ptr(imp), pool.size, chunk, len(imp),
                                  np_ptr(st))
        return st[:n].copy()

    def csc_scatter(self, pool, imp, chunk, staging, dtype=1):
        imp = np.ascontiguousarray(imp, dtype=np.uint8)
        self.L.go_csc_scatter(dtype, np_ptr(pool), np_ptr(imp), pool.size, chunk, len(imp),
                              np_ptr(staging))

    def select_topk(self, norms, k):
        norms = np.ascontiguousarray(norms, dtype=np.float32)
        flags = np.zeros(norms.size, np.uint8)
        self.L.go_select_topk(np_ptr(norms), norms.size, k, np_ptr(flags))
        return flags

    def selection_count(self, s, nc):
        return int(self.L.go_selection_count(s, nc))

    def sparsity_at(self, t, w, s):
        return float(self.L.go_sparsity_at(t, w, s))

    def fnv1a(self, b):
        b = np.ascontiguousarray(b, dtype=np.uint8)
        return int(self.L.go_fnv1a(np_ptr(b), b.size))

    def csc_sgd_update(self, pool, imp, chunk, world, momentum, lr, hu, w, dtype=1):
        imp = np.ascontiguousarray(imp, dtype=np.uint8)
        self.L.go_csc_sgd_update(dtype, np_ptr(pool), np_ptr(imp), pool.size, chunk, len(imp),
                                 world, momentum, lr, np_ptr(hu), np_ptr(w))

    def csc_iteration(self, grads, sizes, chunk, theta, momentum, imp, k_next, hg, dtype=1):
        """One CSC iteration for len(grads) ranks. hg: list of per-rank fp32 arrays (in/out).
        Returns (pools, norms, next_imp, nwin)."""
        n = len(grads)
        s = u64(sizes)
        total = int(s.sum())
        nc = len(imp)
        dt = np.uint16 if dtype == 1 else np.float32
        pools = [np.zeros(total, dt) for _ in range(n)]
        stag = [np.zeros(total, dt) for _ in range(n)]
        norms = [np.zeros(nc, np.float32) for _ in range(n)]
        g = [np.ascontiguousarray(x, dtype=np.float32) for x in grads]
        impa = np.ascontiguousarray(imp, dtype=np.uint8)
        nxt = np.zeros(nc, np.uint8)
        nw = self.L.go_csc_iteration(dtype, n, np_ptr(s), len(s), chunk, theta, momentum,
                                     ptr_array(g), ptr_array(pools), ptr_array(hg),
                                     ptr_array(stag), ptr_array(norms), np_ptr(impa), k_next,
                                     np_ptr(nxt))
        return pools, norms, nxt, nw

    def gen_grads(self, seed, sizes):
        s = u64(sizes)
        out = np.empty(int(s.sum()), np.float32)
        self.L.go_gen_grads(seed, np_ptr(s), len(s), np_ptr(out))
        return out


class Reference:
    """The unmodified reference library (oracle/_ref/libgflowref.so) via ref_driver.cpp."""

    PATH = os.path.join(HERE, "_ref", "libgflowref.so")

    @classmethod
    def available(cls) -> bool:
        return os.path.exists(cls.PATH)

    def __init__(self):
        if not self.available():
            raise RuntimeError("oracle/_ref/libgflowref.so not built (needs /root/reference)")
        L = C.CDLL(self.PATH)
        self.L = L
        L.refd_last_error.restype = C.c_char_p
        L.refd_codec_digest.restype = C.c_uint64
        L.refd_codec_digest.argtypes = [C.c_uint64, C.c_uint64]
        L.refd_selection_count.restype = C.c_uint64
        L.refd_selection_count.argtypes = [C.c_double, C.c_uint64]
        L.refd_sparsity_at.restype = C.c_double
        L.refd_sparsity_at.argtypes = [C.c_uint64, C.c_uint64, C.c_double]
        for name in ["refd_pool_layout", "refd_allreduce", "refd_reduce", "refd_dense_sync", "refd_csc_run",
                     "refd_bench_allreduce", "refd_time_step"]:
            getattr(L, name).restype = C.c_int
        L.refd_time_step.argtypes = [C.c_int, _vp, C.c_int, C.c_uint64, C.c_int, C.c_uint64,
                                     C.c_int, C.c_double, C.c_int, C.c_int, _vp]
        L.refd_f2h_array.argtypes = [_vp, _vp, C.c_uint64]
        L.refd_h2f_array.argtypes = [_vp, _vp, C.c_uint64]
        L.refd_accumulate.argtypes = [C.c_int, _vp, _vp, C.c_uint64]
        L.refd_gen_grads.argtypes = [C.c_int, C.c_int, _vp, C.c_int, _vp]

    def _check(self, rc):
        if rc != 0:
            raise RuntimeError(f"reference error {rc}: {self.L.refd_last_error().decode()}")

    def f2h(self, x):
        x = np.ascontiguousarray(np.asarray(x, dtype=np.float32))
        out = np.empty(x.shape, np.uint16)
        self.L.refd_f2h_array(np_ptr(x), np_ptr(out), x.size)
        return out

    def h2f(self, h):
        h = np.ascontiguousarray(np.asarray(h, dtype=np.uint16))
        out = np.empty(h.shape, np.float32)
        self.L.refd_h2f_array(np_ptr(h), np_ptr(out), h.size)
        return out

    def codec_digest(self, first, count):
        return int(self.L.refd_codec_digest(first, count))

    def accumulate(self, dst, src, dtype=1):
        self.L.refd_accumulate(dtype, np_ptr(dst), np_ptr(src), dst.size)

    def pool_layout(self, sizes, chunk):
        s = u64(sizes)
        off = np.zeros(len(s), np.uint64)
        nc = np.zeros(1, np.uint64)
        cap = int(s.sum() // chunk) + 2
        lens = np.zeros(cap, np.uint64)
        self._check(self.L.refd_pool_layout(np_ptr(s), len(s), C.c_uint64(chunk), np_ptr(off),
                                            np_ptr(nc), np_ptr(lens), C.c_uint64(cap)))
        return off, int(nc[0]), lens[: int(nc[0])].copy()

    def allreduce(self, bufs, dtype=1, algo=0, group_size=1, ring_order=None):
        n = len(bufs)
        sent = np.zeros(n, np.uint64)
        ro = None if ring_order is None else np.ascontiguousarray(ring_order, dtype=np.int32)
        self._check(self.L.refd_allreduce(C.c_int(n), C.c_int(dtype), C.c_uint64(bufs[0].size),
                                          ptr_array(bufs), C.c_int(algo), C.c_int(group_size),
                                          None if ro is None else np_ptr(ro), np_ptr(sent)))
        return sent

    def reduce(self, bufs, root, dtype=1, ring_order=None):
        """The reference's reduce() with ranks as threads, in place; returns payload sent."""
        n = len(bufs)
        sent = np.zeros(n, np.uint64)
        ro = None if ring_order is None else np.ascontiguousarray(ring_order, dtype=np.int32)
        self._check(self.L.refd_reduce(C.c_int(n), C.c_int(dtype), C.c_uint64(bufs[0].size),
                                       ptr_array(bufs), C.c_int(root),
                                       None if ro is None else np_ptr(ro), np_ptr(sent)))
        return sent

    def dense_sync(self, grads, sizes, dtype=1, theta=64 << 20, chunk=32000, algo=0, group_size=1):
        n = len(grads)
        s = u64(sizes)
        total = int(s.sum())
        dt = np.uint16 if dtype == 1 else np.float32
        pools = [np.zeros(total, dt) for _ in range(n)]
        gavg = [np.zeros(total, np.float32) for _ in range(n)]
        g = [np.ascontiguousarray(x, dtype=np.float32) for x in grads]
        cap = len(s) + 2
        wb = np.zeros(cap, np.uint64)
        nw = np.zeros(1, np.uint64)
        sent = np.zeros(n, np.uint64)
        self._check(self.L.refd_dense_sync(
            C.c_int(n), np_ptr(s), C.c_int(len(s)), C.c_uint64(chunk), C.c_int(dtype),
            C.c_uint64(theta), C.c_int(algo), C.c_int(group_size), ptr_array(g), ptr_array(pools),
            ptr_array(gavg), np_ptr(wb), C.c_uint64(cap), np_ptr(nw), np_ptr(sent)))
        return pools, gavg, wb[: int(nw[0])].copy(), sent

    def csc_run(self, grads_steps, sizes, chunk, dtype=1, theta=THETA_INF, final_sparsity=0.9,
                warmup=0, momentum=0.9, lr=0.01, weights0=None, keep=None):
        """grads_steps[t][r] flat ascending. Returns dict of per-step per-rank arrays.
        keep(key, t, r) -> bool selects which outputs to materialise (full-size runs: the
        others are passed as NULL and come back as None); default: all."""
        T, n = len(grads_steps), len(grads_steps[0])
        s = u64(sizes)
        total = int(s.sum())
        _, nc, _ = self.pool_layout(sizes, chunk)
        dt = np.uint16 if dtype == 1 else np.float32
        K = T * n
        if keep is None:
            mk = lambda shape, d: [np.zeros(shape, d) for _ in range(K)]
        else:
            names = iter(["pool_corr", "hg", "pool_x", "norms_loc", "norms_sum", "imp", "next_imp", "hu", "w"])

            def mk(shape, d):
                key = next(names)
                return [np.zeros(shape, d) if keep(key, k // n, k % n) else None for k in range(K)]
        out = dict(pool_corr=mk(total, dt), hg=mk(total, np.float32), pool_x=mk(total, dt),
                   norms_loc=mk(nc, np.float32), norms_sum=mk(nc, np.float32),
                   imp=mk(nc, np.uint8), next_imp=mk(nc, np.uint8), hu=mk(total, np.float32),
                   w=mk(total, np.float32))
        csum = np.zeros(K, np.uint64)
        wins = np.zeros(K, np.uint64)
        g = [np.ascontiguousarray(grads_steps[t][r], dtype=np.float32)
             for t in range(T) for r in range(n)]
        w0 = None if weights0 is None else np.ascontiguousarray(weights0, dtype=np.float32)
        self._check(self.L.refd_csc_run(
            C.c_int(n), np_ptr(s), C.c_int(len(s)), C.c_uint64(chunk), C.c_int(dtype),
            C.c_uint64(theta), C.c_double(final_sparsity), C.c_uint64(warmup),
            C.c_double(momentum), C.c_double(lr), C.c_int(T), ptr_array(g),
            None if w0 is None else np_ptr(w0),
            *[ptr_array(out[k]) for k in ["pool_corr", "hg", "pool_x", "norms_loc", "norms_sum",
                                         "imp", "next_imp", "hu", "w"]],
            np_ptr(csum), np_ptr(wins)))
        res = {k: [[v[t * n + r] for r in range(n)] for t in range(T)] for k, v in out.items()}
        res["checksum"] = csum.reshape(T, n)
        res["windows"] = wins.reshape(T, n)
        return res

    def bench_allreduce(self, ranks, nbytes, algo=0, group_size=1, dtype=0):
        sent, pred = np.zeros(1, np.uint64), np.zeros(1, np.uint64)
        m = np.zeros(1, np.int32)
        self._check(self.L.refd_bench_allreduce(C.c_int(ranks), C.c_uint64(nbytes), C.c_int(algo),
                                                C.c_int(group_size), C.c_int(dtype), np_ptr(sent),
                                                np_ptr(pred), np_ptr(m)))
        return int(sent[0]), int(pred[0]), bool(m[0])

    def gen_grads(self, r, t, sizes):
        s = u64(sizes)
        out = np.empty(int(s.sum()), np.float32)
        self.L.refd_gen_grads(r, t, np_ptr(s), len(s), np_ptr(out))
        return out

    def train(self, ranks=2, model_dims=(64, 32, 1), task="linear", iterations=50, n_examples=1024,
              batch=16, learning_rate=0.01, momentum=0.9, seed=1, algo=0, precision="fp32",
              theta_bytes=64 << 20, csc=False, final_sparsity=0.0, warmup_iters=0, chunk_size=1000):
        d = u64(model_dims)
        nparams = sum(model_dims[i] * model_dims[i - 1] + model_dims[i] for i in range(1, len(model_dims)))
        losses = np.zeros(iterations, np.float64)
        gb = np.zeros(iterations, np.uint64)
        w = np.zeros(nparams, np.float32)
        npo = np.zeros(1, np.uint64)
        self.L.refd_train.restype = C.c_int
        self._check(self.L.refd_train(
            C.c_int(ranks), np_ptr(d), C.c_int(len(d)), C.c_int(task == "logistic"),
            C.c_uint64(iterations), C.c_uint64(n_examples), C.c_uint64(batch), C.c_double(learning_rate),
            C.c_double(momentum), C.c_uint64(seed), C.c_int(algo), C.c_int(precision == "fp16"),
            C.c_uint64(theta_bytes), C.c_int(int(csc)), C.c_double(final_sparsity),
            C.c_uint64(warmup_iters), C.c_uint64(chunk_size), np_ptr(losses), np_ptr(gb), np_ptr(w),
            C.c_uint64(nparams), np_ptr(npo)))
        return dict(loss=losses, grad_payload_bytes=gb, final_weights=w)

    def time_step(self, n, sizes, chunk=32000, dtype=1, theta=64 << 20, csc=False,
                  final_sparsity=0.9, steps=3, warmup=1):
        s = u64(sizes)
        st = np.zeros(5, np.float64)
        self._check(self.L.refd_time_step(n, np_ptr(s), len(s), chunk, dtype, theta, int(csc),
                                          final_sparsity, steps, warmup, np_ptr(st)))
        return dict(zip(["pack", "exchange", "select", "unpack", "total"], st.tolist()))


# Gradient sets (torchvision 0.26 named_parameters(), ascending id).
ALEXNET = [23232, 64, 307200, 192, 663552, 384, 884736, 256, 589824, 256, 37748736, 4096,
           16777216, 4096, 4096000, 1000]
RESNET50 = [
    9408, 64, 64, 4096, 64, 64, 36864, 64, 64, 16384, 256, 256, 16384, 256, 256, 16384, 64, 64,
    36864, 64, 64, 16384, 256, 256, 16384, 64, 64, 36864, 64, 64, 16384, 256, 256, 32768, 128,
    128, 147456, 128, 128, 65536, 512, 512, 131072, 512, 512, 65536, 128, 128, 147456, 128, 128,
    65536, 512, 512, 65536, 128, 128, 147456, 128, 128, 65536, 512, 512, 65536, 128, 128, 147456,
    128, 128, 65536, 512, 512, 131072, 256, 256, 589824, 256, 256, 262144, 1024, 1024, 524288,
    1024, 1024, 262144, 256, 256, 589824, 256, 256, 262144, 1024, 1024, 262144, 256, 256, 589824,
    256, 256, 262144, 1024, 1024, 262144, 256, 256, 589824, 256, 256, 262144, 1024, 1024, 262144,
    256, 256, 589824, 256, 256, 262144, 1024, 1024, 262144, 256, 256, 589824, 256, 256, 262144,
    1024, 1024, 524288, 512, 512, 2359296, 512, 512, 1048576, 2048, 2048, 2097152, 2048, 2048,
    1048576, 512, 512, 2359296, 512, 512, 1048576, 2048, 2048, 1048576, 512, 512, 2359296, 512,
    512, 1048576, 2048, 2048, 2048000, 1000]

# SPDX-License-Identifier: Apache-2.0
"""GradSync: one rank's device-resident gradient-synchronisation step over the C-ABI.

This is the launch sequence a data-parallel trainer runs per iteration, with the
reference's semantics (paths relative to /root/reference/proj):

  dense (lazy allreduce, src/trainer.cpp:297-347 + src/fusion.cpp:72-109):
      gf_pack            all tensors -> fp16 pool in the symmetric heap   (K1)
      gf_ring_allreduce  the FusionEngine theta windows, one launch        (K4)
      gf_unpack          pool -> per-tensor fp32 g_avg = sum * 1/N        (K6)
  CSC (src/sparse.cpp, Algorithm 1):
      gf_csc_pack_correct   pack + residual correction + compaction        (K2)
      gf_ring_allreduce_planned   over the staging buffer                   (K4)
      gf_csc_scatter        staging -> pool (global sums) + exact L1 of those chunks
      (K3 is fused: pack_correct/scatter accumulate exact chunk |x| sums for fp16 pools)
      gf_csc_select         finalize norms, fp32 norm exchange, top-k, next plan (K5)
      gf_csc_sgd_update     unpack + momentum update, important chunks      (K6')

Every launch is asynchronous on the caller's stream; nothing here synchronises or
reads device memory, so a step can be captured into a CUDA graph.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass

from . import capi, cudart

F32, F16 = capi.GF_F32, capi.GF_F16
THETA_INF = capi.THETA_INF


def _align(x: int, a: int = 256) -> int:
    return (x + a - 1) // a * a


def llround_pos(x: float) -> int:
    """C llround for x >= 0 (half away from zero), exact for doubles < 2^52."""
    r = math.floor(x)
    return r + 1 if x - r >= 0.5 else r


@dataclass(frozen=True)
class PoolLayout:
    """GradientPool layout (src/gradient_pool.cpp:11-41): tensor m at offset 0, id 1 last;
    num_chunks = max(1, llround(total / chunk)), the last chunk absorbs the remainder."""

    sizes: tuple
    chunk: int
    offsets: tuple  # offsets[id-1]
    total: int
    num_chunks: int

    @staticmethod
    def build(sizes, chunk=32000) -> "PoolLayout":
        sizes = tuple(int(s) for s in sizes)
        if not sizes:
            raise capi.ConfigError("gradient pool needs at least one tensor")
        if chunk <= 0:
            raise capi.ConfigError("chunk_size must be positive")
        if any(s <= 0 for s in sizes):
            raise capi.ConfigError("tensor sizes must be positive")
        offs = [0] * len(sizes)
        o = 0
        for tid in range(len(sizes), 0, -1):
            offs[tid - 1] = o
            o += sizes[tid - 1]
        nc = max(1, llround_pos(o / chunk))
        return PoolLayout(sizes, chunk, tuple(offs), o, nc)

    def chunk_length(self, c: int) -> int:
        return self.total - c * self.chunk if c + 1 == self.num_chunks else self.chunk


def dense_windows(layout: PoolLayout, esz: int, theta: int):
    """FusionEngine windows of one iteration (src/fusion.cpp:72-109): tensors complete in
    descending id, a window closes when its bytes reach theta, finalize flushes the rest."""
    starts, lens = [], []
    ws = we = 0
    m = len(layout.sizes)
    for tid in range(m, -1, -1):
        flush = tid == 0
        if not flush:
            we = layout.offsets[tid - 1] + layout.sizes[tid - 1]
        hit = theta != THETA_INF and (we - ws) * esz >= theta
        if we > ws and (hit or flush):
            starts.append(ws)
            lens.append(we - ws)
            ws = we
    return starts, lens


def sparsity_at(t: int, warmup: int, final: float) -> float:
    """src/sparse.cpp:13-17"""
    if warmup == 0:
        return final
    return final * min(1.0, t / warmup)


def selection_count(sparsity: float, nc: int) -> int:
    """src/sparse.cpp:19-24 (llround, floor of one chunk)."""
    k = llround_pos((1.0 - sparsity) * nc)
    return max(1, min(k, nc))


class GradSync:
    """Device-resident sync path of one rank. `allgather(bytes) -> list[bytes]` exchanges the
    IPC handles when world > 1 (any control plane: torch.distributed, a TCP store, ...)."""

    def __init__(self, sizes, rank=0, world=1, device=0, dtype=F16, theta=64 << 20,
                 chunk=32000, csc=False, final_sparsity=0.9, warmup_iters=0, momentum=0.9,
                 lr=0.01, allgather=None, timeout_ms=30000, dense_mode="auto", pull_parts=None,
                 csc_mode="push"):
        self.layout = PoolLayout.build(sizes, chunk)
        self.rank, self.world, self.device, self.dtype = rank, world, device, dtype
        self.esz = 2 if dtype == F16 else 4
        self.theta, self.csc = theta, csc
        self.final_sparsity, self.warmup_iters = final_sparsity, warmup_iters
        self.momentum, self.lr = momentum, lr
        L = self.layout
        if dense_mode not in ("auto", "pull", "push", "fused", "rspush"):
            raise capi.ConfigError(f"dense_mode {dense_mode!r}: auto, pull, push, rspush or fused")
        if dense_mode == "auto":
            # measured: the reduce-scatter pushed by the pack is ahead of pull and
            # push-pull at 2 and 4 ranks (ResNet-50 -9 / -8 %, AlexNet -6 / -5 %); fp16 pools only
            dense_mode = "rspush" if dtype == F16 and not csc else ("pull" if world == 2 else "push")
        self.dense_mode = dense_mode
        if csc_mode not in ("pull", "push"):
            raise capi.ConfigError(f"csc_mode {csc_mode!r}: pull or push")
        self.csc_mode = csc_mode
        self.pool_off = 0
        self.stage_off = _align(L.total * self.esz)
        # dense pull mode at N>1: two pools used alternately, so a step never waits for the
        # peers to finish reading the previous step's pool (GF_RSAG_NO_EXIT_BARRIER)
        self._pull_pools = None
        if dense_mode == "pull" and world > 1 and not csc:
            self._pull_pools = [0, self.stage_off]
            self.stage_off += _align(L.total * self.esz)
        self._pull_flip = 0
        # rspush: the pack pushes the reduce-scatter operands into the owners' inboxes
        self._push_inbox = None
        if dense_mode == "rspush" and world > 1 and not csc and self.dtype == F16:
            self._push_inbox = self.stage_off
            self.stage_off += _align((world - 1) * L.total * self.esz)
        # pull mode pieces (units of 1/GF_PART_ONE of every segment): piece k+1 is packed on a
        # side stream while piece k is exchanged; one piece = pack then exchange, serially
        parts = tuple(pull_parts) if pull_parts else (0, capi.GF_PART_ONE)
        if parts[0] != 0 or parts[-1] != capi.GF_PART_ONE or any(a >= b for a, b in zip(parts, parts[1:])):
            raise capi.ConfigError(f"pull_parts {parts!r}: increasing from 0 to {capi.GF_PART_ONE}")
        self.pull_parts = parts
        self._piece_tabs = None
        self._piece_cache = {}
        self._pieces_s = None
        self.norms_off = self.stage_off + (_align(L.total * self.esz) if csc else 0)
        # CSC at N>1: the select's push-inbox (world x nc norms), one barrier instead of two
        self.inbox_off = self.norms_off + _align(L.num_chunks * 4)
        heap = self.inbox_off + (_align(world * L.num_chunks * 4) if csc and world > 1 else 0)
        self.comm = C.c_void_p()
        capi.call("gf_comm_create", world, rank, device, heap, C.byref(self.comm))
        if world > 1:
            if allgather is None:
                raise capi.ConfigError("world > 1 needs an allgather for the IPC handles")
            h = (C.c_char * capi.GF_IPC_HANDLE_BYTES)()
            capi.call("gf_comm_export_handle", self.comm, h)
            handles = allgather(bytes(h))
            capi.call("gf_comm_connect_ipc", self.comm, b"".join(handles))
        capi.call("gf_comm_set_timeout_ms", self.comm, timeout_ms)
        if csc and world > 1:
            capi.call("gf_comm_set_select_inbox", self.comm, self.inbox_off)
        base = C.c_void_p()
        capi.call("gf_comm_heap", self.comm, C.byref(base), None)
        self.heap_base = base.value
        self.pool_ptr = self.heap_base + self.pool_off
        self.last_pool_ptr = self.pool_ptr  # pool that holds the last dense step's sums
        self.stage_ptr = self.heap_base + self.stage_off
        self.norms_ptr = self.heap_base + self.norms_off
        ws, wl = dense_windows(L, self.esz, theta)
        self._win = (capi.u64_array(ws), capi.u64_array(wl), len(ws))
        self._offs = capi.u64_array(L.offsets)
        self._cnts = capi.u64_array(L.sizes)
        self.iteration = 0
        self._csc_bufs = None
        self._side = None  # (stream, event, event) for the CSC update beside the selection
        self._comm_s = None  # (stream, event, event) of the overlapped dense iteration
        self._ov = None

    # ---- state for CSC (allocated by the caller's allocator: torch or cudaMalloc) -------
    def attach_csc_state(self, hg, imp, coff, plan, hu, w, nacc=None):
        """Device buffers: hg (total fp32), imp[2] (nc u8), coff[2] (nc u64), plan[2]
        (4 + nc u64), hu/w (total fp32), nacc (nc u64, zeroed; fp16 pools: exact chunk norms
        fused into pack/scatter). imp[0] must hold iteration 0's set (all ones)."""
        if self.dtype != F16:
            nacc = None
        self._csc_bufs = dict(hg=hg, imp=imp, coff=coff, plan=plan, hu=hu, w=w, nacc=nacc)

    def init_csc_plan(self, stream=None):
        b = self._csc_bufs
        L = self.layout
        capi.call("gf_csc_plan", b["imp"][0], L.total, L.chunk, L.num_chunks, self.dtype,
                  self.theta, b["coff"][0], b["plan"][0], stream)

    # ---- steps ------------------------------------------------------------------------
    @staticmethod
    def _ptrs(ptrs):
        """Per-tensor pointer table; a prebuilt ctypes array is passed through as is."""
        if isinstance(ptrs, C.Array):
            return ptrs
        return (C.c_void_p * len(ptrs))(*ptrs)

    def dense_step(self, grad_ptrs, out_ptrs, stream=None, mark=None, ring_only=False):
        """grad_ptrs/out_ptrs: per-tensor device pointers in ascending tensor id.
        ring_only: diagnostic — the collective alone, on whatever the pool holds."""
        L = self.layout
        m = len(L.sizes)
        mark = mark or (lambda name: None)
        if self.world == 1 and not ring_only:
            # no collective (collectives.cpp:59): gf_sync_step_dense packs and unpacks in one pass
            mark("pack_unpack")
            capi.call("gf_sync_step_dense", self.comm, self.dtype, self.pool_off, self._ptrs(grad_ptrs),
                      self._ptrs(out_ptrs), self._offs, self._cnts, m, self._win[0], self._win[1],
                      self._win[2], stream)
            mark(None)
            return
        if self.world > 1 and self.dense_mode == "fused" and not ring_only:
            return self.fused_step(grad_ptrs, out_ptrs, stream=stream, mark=mark)
        if self._push_inbox is not None and not ring_only:
            self.last_pool_ptr = self.pool_ptr
            mark("push_step")
            capi.call("gf_sync_step_dense_push", self.comm, self.dtype, self.pool_off, self._push_inbox,
                      self._ptrs(grad_ptrs), self._ptrs(out_ptrs), self._offs, self._cnts, m, self._win[0],
                      self._win[1], self._win[2], stream)
            mark(None)
            return
        if self.world > 1 and self.dense_mode == "pull" and not ring_only:
            # pack -> pull reduce-scatter + pull all-gather fused with the unpack
            pool_off, flags = self.pool_off, 0
            if self._pull_pools is not None:
                pool_off = self._pull_pools[self._pull_flip]
                self._pull_flip ^= 1
                flags = capi.GF_RSAG_NO_EXIT_BARRIER
            self.last_pool_ptr = self.heap_base + pool_off
            if len(self.pull_parts) > 2:
                self._pull_pieces(grad_ptrs, out_ptrs, pool_off, flags, stream, mark)
                return
            mark("pack")
            capi.call("gf_pack", self.dtype, self.last_pool_ptr, self._ptrs(grad_ptrs), self._offs,
                      self._cnts, m, 1.0, stream)
            mark("ring_unpack")
            capi.call("gf_ring_allreduce_unpack", self.comm, self.dtype, pool_off, self._ptrs(out_ptrs),
                      self._offs, self._cnts, m, self._win[0], self._win[1], self._win[2], flags, stream)
            mark(None)
            return
        self.last_pool_ptr = self.pool_ptr
        if not ring_only:
            mark("pack")
            capi.call("gf_pack", self.dtype, self.pool_ptr, self._ptrs(grad_ptrs), self._offs,
                      self._cnts, m, 1.0, stream)
        if self.world > 1:  # a world of one has no collective (collectives.cpp:59)
            mark("ring")
            capi.call("gf_ring_allreduce", self.comm, self.dtype, self.pool_off, self._win[0],
                      self._win[1], self._win[2], stream)
        if not ring_only:
            mark("unpack")
            capi.call("gf_unpack", self.dtype, self.pool_ptr, self._ptrs(out_ptrs), self._offs,
                      self._cnts, m, self.world, stream)
        mark(None)

    def _piece_tables(self):
        """Per piece: (tensor index, element offset in the tensor, pool offset, count) of the
        pool ranges the piece covers (gf_part_ranges), cut at tensor boundaries."""
        if self._piece_tabs is None:
            import numpy as np
            L = self.layout
            offs = np.asarray(L.offsets, dtype=np.uint64)
            sizes = np.asarray(L.sizes, dtype=np.uint64)
            ws = [int(x) for x in self._win[0]]
            wl = [int(x) for x in self._win[1]]
            tabs = []
            for lo_q, hi_q in zip(self.pull_parts, self.pull_parts[1:]):
                lo, hi = capi.part_ranges(ws, wl, self.world, lo_q, hi_q)
                ent = []
                for a, b in zip(lo.tolist(), hi.tolist()):
                    for i in np.nonzero((offs < b) & (offs + sizes > a))[0].tolist():
                        s0, s1 = max(a, int(offs[i])), min(b, int(offs[i] + sizes[i]))
                        ent.append((i, s0 - int(offs[i]), s0, s1 - s0))
                tabs.append(np.array(ent, dtype=np.int64).reshape(-1, 4))
            self._piece_tabs = tabs
        return self._piece_tabs

    def _piece_args(self, grad_ptrs):
        """gf_pack tables of every piece for one gradient pointer table (cached per table)."""
        key = id(grad_ptrs) if isinstance(grad_ptrs, C.Array) else tuple(grad_ptrs)
        hit = self._piece_cache.get(key)
        if hit is not None and hit[0] is grad_ptrs:
            return hit[1]
        import numpy as np
        base = np.array([int(p) for p in grad_ptrs], dtype=np.uint64)
        out = []
        for t in self._piece_tables():
            src = base[t[:, 0]] + 4 * t[:, 1].astype(np.uint64)
            out.append(((C.c_void_p * len(t))(*src.tolist()), capi.u64_array(t[:, 2]),
                        capi.u64_array(t[:, 3]), len(t)))
        if len(self._piece_cache) > 64:
            self._piece_cache.clear()
        self._piece_cache[key] = (grad_ptrs, out)
        return out

    def _pull_pieces(self, grad_ptrs, out_ptrs, pool_off, flags, stream, mark):
        """Pull-mode step in pieces: piece 0 is packed and exchanged on `stream` while pieces
        1.. are packed on a side stream; piece k's exchange waits for its pack. Every rank
        launches the pieces' exchanges in the same order (their CTA-pair barriers pair up)."""
        m = len(self.layout.sizes)
        args = self._piece_args(grad_ptrs)
        if self._pieces_s is None:
            cudart.set_device(self.device)
            self._pieces_s = (cudart.stream_create(), cudart.event_create(),
                              [cudart.event_create() for _ in args])
        side, ev_fork, ev_packed = self._pieces_s
        pool = self.heap_base + pool_off
        outp = self._ptrs(out_ptrs)
        mark("pull_step")
        for k, (src, po, cnt, n) in enumerate(args):
            capi.call("gf_pack", self.dtype, pool, src, po, cnt, n, 1.0, stream if k == 0 else side)
            if k == 0:  # the side stream packs the later pieces once piece 0 is packed
                cudart.event_record(ev_fork, stream)
                cudart.stream_wait(side, ev_fork)
            else:
                cudart.event_record(ev_packed[k], side)
        for k in range(len(args)):
            if k > 0:
                cudart.stream_wait(stream, ev_packed[k])
            capi.call("gf_ring_allreduce_unpack_part", self.comm, self.dtype, pool_off, outp, self._offs,
                      self._cnts, m, self._win[0], self._win[1], self._win[2], self.pull_parts[k],
                      self.pull_parts[k + 1], flags, stream)
        mark(None)

    def fused_step(self, grad_ptrs, out_ptrs, stream=None, mark=None):
        """The dense step as ONE kernel (gf_sync_step_dense): pack, NVLink ring of the theta
        windows and unpack overlapped slab by slab; bit-identical to dense_step."""
        mark = mark or (lambda name: None)
        mark("fused_step")
        capi.call("gf_sync_step_dense", self.comm, self.dtype, self.pool_off, self._ptrs(grad_ptrs),
                  self._ptrs(out_ptrs), self._offs, self._cnts, len(self.layout.sizes),
                  self._win[0], self._win[1], self._win[2], stream)
        mark(None)

    # ---- overlap with backward: FusionEngine on device streams (fusion.cpp:25-123) --------
    def begin_iteration(self, grad_ptrs, out_ptrs, stream=None):
        """Start a dense iteration whose tensors become final one by one (descending id)
        while the caller's backward is still running on `stream`. Each theta window is
        packed, ring-reduced and unpacked on a communication stream as soon as it closes
        (maybe_launch, fusion.cpp:72-99), FIFO like the reference's progress thread."""
        if self.dtype not in (F16, F32):
            raise capi.ConfigError("bad dtype")
        self._ov = dict(grad=list(grad_ptrs), out=list(out_ptrs), stream=stream, ws=0, we=0,
                        ids=[], launched=0)

    def tensor_complete(self, tid):
        """FusionEngine::on_tensor_complete(tid) (fusion.cpp:72-99); tid is 1-based and
        tensors complete in descending id order (the pool's ascending offsets)."""
        ov = self._ov
        L = self.layout
        if ov is None:
            raise capi.ConfigError("tensor_complete before begin_iteration")
        expect = len(L.sizes) - len(ov["ids"]) - ov["launched"]
        if tid != expect:
            raise capi.ConfigError(f"tensor {tid} completed out of order (expected {expect})")
        ov["ids"].append(tid)
        ov["we"] = L.offsets[tid - 1] + L.sizes[tid - 1]
        if self.theta != THETA_INF and (ov["we"] - ov["ws"]) * self.esz >= self.theta:
            self._launch_window()

    def finalize_iteration(self):
        """finalize_iteration + wait_all (fusion.cpp:101-123): flush the last window and make
        the caller's stream wait for every window's g_avg."""
        ov = self._ov
        if ov is None:
            raise capi.ConfigError("finalize_iteration before begin_iteration")
        if ov["we"] > ov["ws"]:
            self._launch_window()
        if ov["launched"] != len(self.layout.sizes):
            raise capi.ConfigError("finalize_iteration before every tensor completed")
        cs, ev_ready, ev_done = self._comm_stream()
        cudart.stream_wait(ov["stream"], ev_done)
        self._ov = None

    def _launch_window(self):
        ov = self._ov
        cs, ev_ready, ev_done = self._comm_stream()
        ids = ov["ids"]
        n = len(ids)
        src = (C.c_void_p * n)(*[ov["grad"][t - 1] for t in ids])
        dst = (C.c_void_p * n)(*[ov["out"][t - 1] for t in ids])
        offs = capi.u64_array([self.layout.offsets[t - 1] for t in ids])
        cnts = capi.u64_array([self.layout.sizes[t - 1] for t in ids])
        cudart.event_record(ev_ready, ov["stream"])  # the window's gradients are final
        cudart.stream_wait(cs, ev_ready)
        ws, wl = capi.u64_array([ov["ws"]]), capi.u64_array([ov["we"] - ov["ws"]])
        if self.world == 1:
            capi.call("gf_sync_step_dense", self.comm, self.dtype, self.pool_off, src, dst, offs, cnts,
                      n, ws, wl, 1, cs)
        else:
            capi.call("gf_pack", self.dtype, self.pool_ptr, src, offs, cnts, n, 1.0, cs)
            capi.call("gf_ring_allreduce", self.comm, self.dtype, self.pool_off, ws, wl, 1, cs)
            capi.call("gf_unpack", self.dtype, self.pool_ptr, dst, offs, cnts, n, self.world, cs)
        cudart.event_record(ev_done, cs)
        ov["launched"] += n
        ov["ids"] = []
        ov["ws"] = ov["we"]

    def _comm_stream(self):
        if self._comm_s is None:
            cudart.set_device(self.device)
            self._comm_s = (cudart.stream_create(), cudart.event_create(), cudart.event_create())
        return self._comm_s

    def csc_step(self, grad_ptrs, stream=None, mark=None):
        """One CSC iteration (Algorithm 1). Uses the buffers given to attach_csc_state."""
        b = self._csc_bufs
        L = self.layout
        m = len(L.sizes)
        cur, nxt = self.iteration & 1, (self.iteration + 1) & 1
        marked = mark is not None
        mark = mark or (lambda name: None)
        mark("pack_correct")
        nacc = b["nacc"]
        solo = self.world == 1  # the exchange is the identity: no staging, no scatter
        capi.call("gf_csc_pack_correct", self.dtype, self.pool_ptr, b["hg"],
                  None if solo else self.stage_ptr, b["imp"][cur], b["coff"][cur], L.total, L.chunk,
                  L.num_chunks, self._ptrs(grad_ptrs), self._offs, self._cnts, m, self.momentum,
                  nacc, stream)
        # chunks selected for this iteration (iteration 0 is dense, sparse.cpp:45-51)
        k_cur = L.num_chunks if self.iteration == 0 else selection_count(
            sparsity_at(self.iteration, self.warmup_iters, self.final_sparsity), L.num_chunks)
        fused_wb = not solo and nacc is not None and L.chunk % 8 == 0 and L.num_chunks <= 6144
        if fused_wb and self.csc_mode == "pull":
            # pull RS + pull AG straight into the pool (+ exact L1); the staging buffer is next
            # rewritten after gf_csc_select's barrier, so no exit barrier is needed
            mark("ring_scatter")
            capi.call("gf_csc_exchange_pull", self.comm, self.stage_off, b["plan"][cur], self.pool_ptr,
                      L.chunk, L.num_chunks, nacc, stream)
        elif fused_wb:  # exchange + write-back + exact L1 of the exchanged chunks, one launch
            mark("ring_scatter")
            capi.call("gf_ring_allreduce_planned_scatter", self.comm, self.dtype, self.stage_off,
                      b["plan"][cur], self.pool_ptr, L.chunk, L.num_chunks, nacc, stream)
        elif not solo:
            mark("ring")
            capi.call("gf_ring_allreduce_planned", self.comm, self.dtype, self.stage_off,
                      b["plan"][cur], stream)
        if not solo and not fused_wb:
            mark("scatter")
            capi.call("gf_csc_scatter", self.dtype, self.pool_ptr, self.stage_ptr, b["plan"][cur],
                      b["coff"][cur], L.total, L.chunk, L.num_chunks, k_cur, nacc, stream)
        if nacc is None:  # fp32 pool: separate norm pass (sequential fp64, as the reference)
            mark("norms")
            capi.call("gf_chunk_norms", self.dtype, self.pool_ptr, L.total, L.chunk, L.num_chunks,
                      b["imp"][cur], self.world, self.norms_ptr, stream)
        k = selection_count(sparsity_at(self.iteration + 1, self.warmup_iters,
                                        self.final_sparsity), L.num_chunks)

        def select():
            capi.call("gf_csc_select", self.comm, self.norms_off, L.num_chunks, k, b["imp"][nxt],
                      L.total, L.chunk, self.dtype, self.theta, b["coff"][nxt], b["plan"][nxt],
                      nacc, self.pool_ptr if nacc else None, b["imp"][cur] if nacc else None, stream)

        def update(s):
            capi.call("gf_csc_sgd_update", self.dtype, self.pool_ptr, b["plan"][cur], L.total,
                      L.chunk, L.num_chunks, k_cur, self.world, self.momentum, self.lr, b["hu"],
                      b["w"], s)

        if marked:  # per-kernel timing: one stream, kernels in order
            mark("select")
            select()
            mark("sgd_update")
            update(stream)
        else:
            # The update reads this iteration's pool and plan; the selection reads the
            # pool and writes the NEXT plan and norms: independent. The one-CTA, latency-bound
            # selection runs beside the bandwidth-bound update on a second stream; the step
            # ends when both did (the next pack_correct overwrites the pool).
            side, ev_a, ev_b = self._side_stream()
            cudart.event_record(ev_a, stream)
            cudart.stream_wait(side, ev_a)
            update(side)
            cudart.event_record(ev_b, side)
            select()
            cudart.stream_wait(stream, ev_b)
        mark(None)
        self.iteration += 1

    def _side_stream(self):
        if self._side is None:
            cudart.set_device(self.device)
            self._side = (cudart.stream_create(), cudart.event_create(), cudart.event_create())
        return self._side

    def status(self):
        capi.call("gf_comm_status", self.comm)

    def close(self):
        if self.comm:
            capi.call("gf_comm_destroy", self.comm)
            self.comm = C.c_void_p()

# SPDX-License-Identifier: Apache-2.0
"""Benchmark of the B200 gradient-sync path (GradientFlow, arXiv 1902.06855).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload NAME] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...      (one process per GPU, NCCL plumbing)

A step = one data-parallel gradient synchronisation of one iteration's gradients:
dense: pack (fp32 -> fp16 pool) + NVLink ring allreduce of the theta windows + unpack
(g_avg = sum/N per tensor); CSC: pack+correct+compact, ring over the staging buffer,
write-back, exact chunk L1, norm exchange + top-k, unpack+momentum update.
Prints ONE JSON line (rank 0). See DESIGN.md for the roofline accounting.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

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
THETA_INF = (1 << 64) - 1
L2_BYTES = 126 << 20

WORKLOADS = {
    # BASELINE.json configs[1]: ResNet-50 gradient set, dense lazy allreduce, fp16 wire.
    "resnet50-dense": dict(sizes=RESNET50, model="resnet50", csc=False, theta=64 << 20),
    "alexnet-dense": dict(sizes=ALEXNET, model="alexnet", csc=False, theta=64 << 20),
    # configs[2]: AlexNet CSC, chunk 32000, keep top 10% by norm, residual accumulation.
    "alexnet-csc": dict(sizes=ALEXNET, model="alexnet", csc=True, theta=THETA_INF, sparsity=0.9),
    # configs[3]: ResNet-50 CSC with a lazy-fusion threshold (sweep via --theta).
    "resnet50-csc": dict(sizes=RESNET50, model="resnet50", csc=True, theta=64 << 20, sparsity=0.9),
}


def env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """SM clocks + throttle reasons while the timed work executes.

    sample_now() is called by the main thread right after the timed steps are enqueued
    (the GPU is still executing them) — no sampling thread competes for the GIL with the
    launch loop. A separate nvidia-smi process (-lms 50) records the whole run for reasons."""

    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
               0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, device_index):
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self.proc = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None
        try:
            import subprocess
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={device_index}",
                 "--query-gpu=clocks.sm,clocks_event_reasons.hw_slowdown,"
                 "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                 "clocks_event_reasons.sw_power_cap", "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def sample_now(self):
        if self.nv is None:
            return
        try:
            self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
            r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            for bit, name in self.REASONS.items():
                if r & bit:
                    self.reasons.add(name)
        except Exception:
            pass

    def stop(self):
        smi = 0
        if self.proc is not None:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
                names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
                for line in out.splitlines():
                    f = [x.strip() for x in line.split(",")]
                    if len(f) != 5:
                        continue
                    smi += 1
                    for name, v in zip(names, f[1:]):
                        if v.lower() == "active":
                            self.reasons.add(name)
            except Exception:
                pass
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples), "smi_samples_whole_run": smi}


def ring_bus_bytes(layout, esz, world, windows):
    """NCCL busBw convention: 2(N-1)/N * K per rank (K = window bytes)."""
    if world == 1:
        return 0
    return sum(2 * (world - 1) * (wl * esz) / world for wl in windows)


def reference_arm(args, wl, world, rank):
    """--impl reference: the reference's own CPU implementation (oracle/_ref, unmodified
    library compiled from /root/reference) on the host cores, ranks as threads."""
    if rank != 0:
        return 0
    from oracle.oracle import Reference
    ref = Reference()
    steps = max(1, args.steps)
    st = ref.time_step(world, wl["sizes"], chunk=32000, dtype=1, theta=wl["theta"],
                       csc=wl["csc"], final_sparsity=wl.get("sparsity", 0.9), steps=steps,
                       warmup=max(1, args.warmup if args.warmup < 3 else 1))
    line = {
        "metric": "grad-sync ms/step", "value": round(st["total"], 3), "unit": "ms",
        "n_gpus": world, "steps": steps, "warmup": args.warmup, "ms_per_step": round(st["total"], 3),
        "higher_is_better": False, "scaling": "weak", "vs_baseline": None, "dtype": "fp16",
        "data": "synthetic", "impl": "reference",
        "config": config_of(args, wl, world),
        "stages_ms": {k: round(v, 3) for k, v in st.items()},
        "cpu_baseline": {"value": round(st["total"], 3), "unit": "ms", "cores": world,
                         "kind": "reference",
                         "sample": f"{steps} timed steps (+1 warm-up) of the full workload, "
                                   f"{world} rank thread(s) over InprocTransport"},
        "e2e": {"value": round(st["total"], 3), "unit": "ms", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def config_of(args, wl, world):
    theta = wl["theta"]
    return {"workload": args.workload, "gradient_set": wl["model"],
            "tensors": len(wl["sizes"]), "elements": sum(wl["sizes"]),
            "wire": "fp16", "chunk": 32000,
            "theta_bytes": "inf" if theta == THETA_INF else theta,
            "csc_sparsity": wl.get("sparsity") if wl["csc"] else None,
            "parallelism": f"dp{world}", "global_batch": None, "seq_len": None}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--workload", default="resnet50-dense", choices=sorted(WORKLOADS))
    ap.add_argument("--theta", type=int, default=None, help="override theta bytes (-1 = inf)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--trace", action="store_true", help="report ring CTA-0 timestamps (diagnostic)")
    ap.add_argument("--overlap", type=float, default=0.0, metavar="BACKWARD_MS",
                    help="also measure the dense sync overlapped with a synthetic backward of "
                         "this many ms (bf16 GEMMs; tensors complete in descending id, theta "
                         "windows launch as they close: the reference's lazy allreduce)")
    ap.add_argument("--dense-mode", default="auto", choices=["auto", "pull", "push", "rspush"],
                    help="dense N>1: rspush (pack pushes the reduce-scatter operands to their owners, "
                         "local reduce + all-gather push, unpack), pull (pack + pull RS/AG fused with "
                         "unpack), push (pack + push-pull ring + unpack); auto = rspush")
    ap.add_argument("--csc-mode", default="push", choices=["pull", "push"],
                    help="CSC N>1 exchange: pull (pull RS/AG straight into the pool) or push "
                         "(push-pull ring + fused write-back)")
    args = ap.parse_args()

    wl = dict(WORKLOADS[args.workload])
    if args.theta is not None:
        wl["theta"] = THETA_INF if args.theta < 0 else args.theta
    world = env_int("WORLD_SIZE", 1)
    rank = env_int("RANK", 0)
    local = env_int("LOCAL_RANK", 0)
    if args.impl == "reference":
        return reference_arm(args, wl, world, rank)

    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_1902_06855_b200 import capi
    from paper_1902_06855_b200.engine import GradSync, dense_windows

    torch.cuda.set_device(local)
    from paper_1902_06855_b200 import cudart
    cudart.set_device(local)  # the library's CUDA runtime (may differ from torch's) on the same GPU
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    def allgather(b):
        out = [None] * world
        dist.all_gather_object(out, b)
        return out

    sizes = wl["sizes"]
    csc = wl["csc"]
    sync = GradSync(sizes, rank=rank, world=world, device=local, theta=wl["theta"], csc=csc,
                    final_sparsity=wl.get("sparsity", 0.9), allgather=allgather,
                    dense_mode=args.dense_mode, csc_mode=args.csc_mode)
    L = sync.layout
    total = L.total
    esz = 2
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream()
    sp = stream.cuda_stream

    # ---- synthetic gradients: rotating input sets so every step reads inputs not in L2 ------
    in_bytes = total * 4
    n_sets = max(2, math.ceil(2 * L2_BYTES / in_bytes) + 1)
    g = torch.Generator(device=dev)
    g.manual_seed(1234 + rank)
    scales = torch.cat([torch.full((s,), 2.0 ** -((i + 1) % 7), device=dev) for i, s in enumerate(sizes)])
    inputs = [(torch.rand(total, device=dev, generator=g) * 2 - 1) * scales for _ in range(n_sets)]
    bounds = np.concatenate([[0], np.cumsum(sizes)])

    def views(flat):
        return [flat[int(bounds[i]):int(bounds[i + 1])].data_ptr() for i in range(len(sizes))]

    import ctypes as C
    in_ptrs = [(C.c_void_p * len(sizes))(*views(x)) for x in inputs]  # prebuilt launch tables
    outs = [torch.empty(total, device=dev) for _ in range(2)]
    out_ptrs = [(C.c_void_p * len(sizes))(*views(x)) for x in outs]
    def step(i):
        if csc:
            sync.csc_step(in_ptrs[i % n_sets], stream=sp)
        else:
            sync.dense_step(in_ptrs[i % n_sets], out_ptrs[i % 2], stream=sp)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    clocks = ClockSampler(local)
    warm = max(args.warmup, 0)
    for i in range(warm):
        step(i)
    barrier()
    launches0 = capi.lib().gf_kernel_launches()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    barrier()
    t0.record(stream)
    h0 = time.perf_counter()
    for i in range(args.steps):
        step(warm + i)
    t1.record(stream)
    host_enqueue_ms = (time.perf_counter() - h0) * 1e3 / max(args.steps, 1)
    clocks.sample_now()  # the GPU is still executing the queued timed steps here
    torch.cuda.synchronize()
    barrier()
    launches = capi.lib().gf_kernel_launches() - launches0
    sync.status()
    ms_local = t0.elapsed_time(t1) / max(args.steps, 1)

    # per-kernel durations: the same K steps again, with CUDA events on the launching stream
    # between the kernels. Kept out of the headline pass: an event between two kernels costs
    # the step ~3-4 us of GPU time (scripts/hbm_probe.py), so `kernels` is slightly pessimistic.
    sync.set_marks(True)
    for i in range(args.steps):
        step(warm + args.steps + i)
    torch.cuda.synchronize()
    seg_ms = sync.marks()
    sync.set_marks(False)
    barrier()
    sync.status()

    def allmax(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    ms = allmax(ms_local)
    seg_ms = {k: allmax(v) for k, v in sorted(seg_ms.items())}
    kernel_timing = "events between kernels, second pass of the same K steps"
    if len(seg_ms) == 1 and launches == args.steps:
        # one launch per step: the headline pass's t0/t1 events over K back-to-back launches
        # ARE that kernel's average launch duration, without per-kernel event overhead
        seg_ms = {k: ms for k in seg_ms}
        kernel_timing = "one launch per step: t0/t1 events over the K timed launches"

    # ---- roofline of the dominant kernel ------------------------------------------------
    hbm_peak, peak_src = load_peaks()
    ws, wlen = dense_windows(L, esz, wl["theta"])
    algo = {  # algorithmic bytes per launch
        "pack": total * 6, "unpack": total * 6, "pack_correct": total * 14,
        "pack_unpack": total * 10,  # N=1: g in (4), pool out (2), g_avg out (4)
        "norms": total * 2, "scatter": None, "select": None, "sgd_update": None,
        "ring": None,
    }
    if csc:
        # staged elements of the last timed (sparse) iteration, read back after timing
        pc = np.zeros(1, np.uint64)
        cudart.memcpy(pc.ctypes.data, sync.state("plan_cur")[0], 8)
        cudart.sync_device()
        staged = int(pc[0])
        # g, hg in; pool, hg out; + the staging copy at N>1 (N=1 has no exchange, no staging)
        algo["pack_correct"] = total * 14 + (staged * 2 if world > 1 else 0)
        algo["scatter"] = staged * 4                      # staging in, pool out (+ exact L1)
        algo["sgd_update"] = staged * 18                  # pool in; hu, w in+out
        ring_bytes = ring_bus_bytes(L, esz, world, [staged])
    else:
        ring_bytes = ring_bus_bytes(L, esz, world, wlen)
    algo["ring"] = ring_bytes if world > 1 else None
    algo["ring_scatter"] = algo["ring"]  # CSC exchange with the write-back fused in
    algo["ring_unpack"] = algo["ring"]   # dense pull mode: RS + AG with the unpack fused in
    algo["rsp"] = algo["ring"]           # rspush: local reduce + all-gather push (the NVLink kernel)
    algo["pack_push"] = total * 6        # rspush: the routed pack (HBM 6 B/el; its NVLink stores ride on it)
    dom = max(seg_ms, key=lambda k: seg_ms[k]) if seg_ms else None
    roof = None
    if dom is not None and algo.get(dom):
        t_s = seg_ms[dom] / 1e3
        if dom in ("ring", "ring_scatter", "ring_unpack", "rsp"):
            ach = algo[dom] / t_s / 1e9
            roof = {"bound": "nvlink", "achieved": round(ach, 1), "peak": 900.0, "unit": "GB/s",
                    "frac": round(ach / 900.0, 3), "traffic": None,
                    "kernel": "ring_kernel" if dom == "ring" else dom,
                    "peak_src": "NVLink 5 nominal 900 GB/s/direction (measured peer copy 770)",
                    "frac_of_measured_770": round(ach / 770.0, 3)}
            if dom == "ring_unpack":
                roof["note"] = "the unpack HBM pass sits inside the time the NVLink bus bytes are divided by"
        else:
            ach = algo[dom] / t_s / 1e9
            roof = {"bound": "hbm", "achieved": round(ach, 1), "peak": hbm_peak, "unit": "GB/s",
                    "frac": round(ach / hbm_peak, 3), "traffic": None, "kernel": dom,
                    "peak_src": peak_src}
    # traffic: DRAM bytes per launch of the dominant kernel from the committed ncu capture
    if roof is not None:
        try:
            with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
                tr = json.load(f)
            kname = {"pack": "pack_kernel", "pack_unpack": "pack_kernel", "unpack": "unpack_kernel", "pack_correct": "pack_correct_kernel",
                     "sgd_update": "csc_sgd_kernel", "scatter": "compact_kernel",
                     "select": "select_kernel", "pack_push": "pack_push_kernel", "rsp": "rsp_kernel"}.get(dom)
            ent = tr.get(args.workload, {}).get(kname or "", {})
            if ent:
                roof["traffic"] = ent["dram_bytes_per_launch"]
                roof["traffic_note"] = "ncu --set full, cold cache, profiles/ncu_traffic.json"
        except Exception:
            pass
    kernels = {}
    for k, v in seg_ms.items():
        d = {"ms": round(v, 4)}
        if algo.get(k):
            d["GBps"] = round(algo[k] / (v / 1e3) / 1e9, 1)
            if k not in ("ring", "ring_scatter", "ring_unpack", "rsp"):
                d["frac_hbm"] = round(d["GBps"] / hbm_peak, 3)
            else:
                d["busbw_frac_900"] = round(d["GBps"] / 900, 3)
        kernels[k] = d

    # ---- ring trace (diagnostic, outside the timed region): device timestamps of CTA 0 ----
    ring_trace = None
    if args.trace and world > 1:
        import ctypes as _C
        capi.call("gf_comm_set_trace", sync.comm, 1)
        rec = []
        for i in range(args.steps):
            barrier()
            step(i)
            torch.cuda.synchronize()
            t = (_C.c_uint64 * 11)()
            capi.call("gf_comm_trace_n", sync.comm, t, 11)
            rec.append([t[1] - t[0], t[2] - t[1], t[3] - t[2]] +
                       ([t[5] - t[4], t[6] - t[5], t[7] - t[6], t[8] - t[7], t[9] - t[8], t[10] - t[9]]
                        if csc else []))
        capi.call("gf_comm_set_trace", sync.comm, 0)
        med = [statistics.median(r[j] for r in rec) / 1e3 for j in range(3)]  # ring CTA 0
        ring_trace = {"entry_wait_us": round(allmax(med[0]), 2), "body_us": round(allmax(med[1]), 2),
                      "exit_wait_us": round(allmax(med[2]), 2)}
        per_rank = [None] * world
        dist.all_gather_object(per_rank, [round(m, 2) for m in med])
        ring_trace["per_rank_entry_body_exit_us"] = per_rank
        if csc:  # gf_csc_select phases (thread 0): finalize, entry wait, ring-order sums, exit wait, top-k, plan
            ring_trace["select_phases_us"] = [round(allmax(statistics.median(r[j] for r in rec) / 1e3), 2)
                                              for j in range(3, 9)]

    # ---- overlap with backward (fusion.cpp:72-123) -----------------------------
    overlap = None
    if args.overlap > 0 and not csc:
        A = torch.randn(2048, 4096, dtype=torch.bfloat16, device=dev)
        B = torch.randn(4096, 4096, dtype=torch.bfloat16, device=dev)
        Cm = torch.empty(2048, 4096, dtype=torch.bfloat16, device=dev)
        for _ in range(20):
            torch.matmul(A, B, out=Cm)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(50):
            torch.matmul(A, B, out=Cm)
        e1.record(stream)
        torch.cuda.synchronize()
        gemm_ms = e0.elapsed_time(e1) / 50
        n_gemm = max(1, round(args.overlap / gemm_ms))
        # backward work of tensor id is proportional to its size (tiny BN tensors: none)
        reps = {tid: int(round(n_gemm * sizes[tid - 1] / total)) for tid in range(1, len(sizes) + 1)}

        def backward(i, with_sync):
            if with_sync:
                sync.begin_iteration(in_ptrs[i % n_sets], out_ptrs[i % 2], stream=sp)
            for tid in range(len(sizes), 0, -1):
                for _ in range(reps[tid]):
                    torch.matmul(A, B, out=Cm)
                if with_sync:
                    sync.tensor_complete(tid)
            if with_sync:
                sync.finalize_iteration()

        # Alternate the two variants step by step and take medians: GEMM throughput drifts
        # by several % over a run (power, clocks), more than the sync itself at N=1.
        for i in range(3):
            backward(i, False)
            backward(i, True)
        barrier()
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(2 * args.steps + 1)]
        h0 = time.perf_counter()
        evs[0].record(stream)
        for i in range(args.steps):
            backward(i, False)
            evs[2 * i + 1].record(stream)
            backward(i, True)
            evs[2 * i + 2].record(stream)
        host_ms = (time.perf_counter() - h0) * 1e3 / max(args.steps, 1)
        torch.cuda.synchronize()
        barrier()
        t_bw = [evs[2 * i].elapsed_time(evs[2 * i + 1]) for i in range(args.steps)]
        t_both = [evs[2 * i + 1].elapsed_time(evs[2 * i + 2]) for i in range(args.steps)]
        bw = allmax(statistics.median(t_bw))
        both = allmax(statistics.median(t_both))
        overlap = {"backward_ms": round(bw, 4), "backward_plus_sync_ms": round(both, 4),
                   "exposed_sync_ms": round(both - bw, 4), "sync_alone_ms": round(ms, 4),
                   "windows": len(wlen), "theta_bytes": "inf" if wl["theta"] == THETA_INF else wl["theta"],
                   "host_enqueue_ms_per_pair": round(host_ms, 4),
                   "method": "backward-only and backward+sync steps alternate; medians, max over ranks",
                   "backward": f"{sum(reps.values())} bf16 GEMMs 2048x4096x4096 per step, by tensor size"}

    # ---- NCCL allreduce on the same fp16 volume (comparison only) ---------------------------
    nccl = None
    if world > 1:
        x = torch.zeros(total, dtype=torch.float16, device=dev)
        for _ in range(3):
            dist.all_reduce(x)
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            dist.all_reduce(x)
        e1.record(stream)
        torch.cuda.synchronize()
        nms = allmax(e0.elapsed_time(e1) / max(args.steps, 1))
        nccl = {"ms": round(nms, 4), "busbw_GBps": round(2 * (world - 1) / world * total * 2 / (nms / 1e3) / 1e9, 1)}

    # ---- end-to-end through the C-ABI with host buffers ---------------------------------------
    e2e = None
    if not args.no_e2e:
        # Every step: H2D of the step's gradients from pinned host memory, the sync step
        # through the C-ABI, D2H of its result (g_avg, or the updated weights for CSC).
        # Double-buffered on three streams, as a training loop would run it: the H2D of
        # step i+1 overlaps the D2H of step i (PCIe is full duplex); a step starts once its
        # input landed and the previous result left the device (CSC updates w in place).
        h_in = [torch.empty(total, dtype=torch.float32, pin_memory=True) for _ in range(2)]
        for h in h_in:
            h.copy_(inputs[0].cpu())
        h_out = [torch.empty(total, dtype=torch.float32, pin_memory=True) for _ in range(2)]
        d2h = total * 4
        s_in, s_out = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)

        wptr = sync.state("w")[0] if csc else None

        def run_e2e(k):
            ev_in = [torch.cuda.Event() for _ in range(k)]
            ev_comp = [torch.cuda.Event() for _ in range(k)]
            ev_out = [torch.cuda.Event() for _ in range(k)]
            for i in range(k):
                slot = i % 2
                if i >= 2:
                    s_in.wait_event(ev_comp[i - 2])  # step i-2 finished reading this input slot
                with torch.cuda.stream(s_in):
                    inputs[slot].copy_(h_in[slot], non_blocking=True)
                ev_in[i].record(s_in)
                stream.wait_event(ev_in[i])
                if i >= 1:
                    stream.wait_event(ev_out[i - 1])
                step(slot)
                ev_comp[i].record(stream)
                s_out.wait_event(ev_comp[i])
                if csc:  # the updated weights w (engine-owned) leave the device
                    cudart.memcpy(h_out[slot].data_ptr(), wptr, d2h, s_out.cuda_stream)
                else:
                    with torch.cuda.stream(s_out):
                        h_out[slot].copy_(outs[slot], non_blocking=True)
                ev_out[i].record(s_out)
            return ev_out[-1]

        run_e2e(3)
        torch.cuda.synchronize()
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(s_in)
        stream.wait_event(e0)
        last = run_e2e(args.steps)
        s_out.wait_event(last)
        e1.record(s_out)
        torch.cuda.synchronize()
        ems = allmax(e0.elapsed_time(e1) / max(args.steps, 1))
        e2e = {"value": round(ems, 4), "unit": "ms", "h2d_bytes_per_step": total * 4,
               "d2h_bytes_per_step": d2h,
               "path": "C-ABI gf_* with pinned host grads in / results out, double-buffered: "
                       "H2D of step i+1 overlaps D2H of step i"}
    sync.status()

    clk = clocks.stop()
    cpu = None
    if world == 1 and rank == 0 and not args.no_cpu_baseline:
        try:
            from oracle.oracle import Reference
            if Reference.available():
                st = Reference().time_step(1, sizes, chunk=32000, dtype=1, theta=wl["theta"],
                                           csc=csc, final_sparsity=wl.get("sparsity", 0.9),
                                           steps=3, warmup=1)
                cpu = {"value": round(st["total"], 3), "unit": "ms", "cores": 1, "kind": "reference",
                       "sample": "3 timed steps (+1 warm-up) of the full workload, 1 rank thread",
                       "stages_ms": {k: round(v, 2) for k, v in st.items()}}
        except Exception as e:  # pragma: no cover
            cpu = {"error": str(e)[:200]}

    if rank == 0:
        bus = None
        rk = next((k for k in ("ring", "ring_unpack", "ring_scatter", "rsp") if k in seg_ms), "ring")
        if world > 1 and rk in seg_ms:
            bus = round(ring_bytes / (seg_ms[rk] / 1e3) / 1e9, 1)
        line = {
            "metric": "grad-sync ms/step", "value": round(ms, 4), "unit": "ms", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4),
            "higher_is_better": False, "scaling": "weak", "vs_baseline": None, "dtype": "fp16",
            "data": "synthetic", "config": dict(config_of(args, wl, world),
                                                exchange=("none (N=1)" if world == 1 else
                                                          (sync.csc_mode if csc else sync.dense_mode)),
                                                l2=f"{n_sets} rotating input sets of {in_bytes >> 20} MiB "
                                                   f"(> 126 MB L2)"),
            "bus_gbs": bus, "kernels": kernels, "kernel_timing": kernel_timing, "roofline": roof, "cpu_baseline": cpu, "e2e": e2e,
            "nccl_allreduce": nccl, "gpu_launches": int(launches), "clocks": clk,
            "ring_trace": ring_trace, "overlap": overlap, "host_enqueue_ms_per_step": round(host_enqueue_ms, 4),
        }
        print(json.dumps(line), flush=True)
    sync.close()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())

# SPDX-License-Identifier: Apache-2.0
"""Benchmark of the B200 gradient-sync path (GradientFlow, arXiv 1902.06855).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload NAME] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...      (one process per GPU, NCCL plumbing)

A step = one data-parallel gradient synchronisation of one iteration's gradients through the
native engine (gf_engine_*): dense = pack (fp32 -> fp16 pool) + NVLink allreduce of the theta
windows + unpack (g_avg = sum/N per tensor); CSC = pack+correct+compact, exchange + write-back
+ exact chunk L1, norm exchange + top-k, momentum update of the important chunks.
Inputs are SURVEY.md §8(d)'s seeded gradients (std::mt19937_64(1234 + rank + 7919 t), the
stream the reference arm draws too). Prints ONE JSON line (rank 0): the headline workload,
plus a `csc` sub-object for the CSC workload (AlexNet, configs[2]). See DESIGN.md §7.
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
NVLINK_GBS = 900.0

WORKLOADS = {
    # BASELINE.json configs[1]: ResNet-50 gradient set, dense lazy allreduce, fp16 wire.
    "resnet50-dense": dict(sizes=RESNET50, model="resnet50", csc=False, theta=64 << 20),
    "alexnet-dense": dict(sizes=ALEXNET, model="alexnet", csc=False, theta=64 << 20),
    # configs[2]: AlexNet CSC, chunk 32000, keep top 10% by norm, residual accumulation.
    "alexnet-csc": dict(sizes=ALEXNET, model="alexnet", csc=True, theta=THETA_INF, sparsity=0.9),
    # configs[3]: ResNet-50 CSC with a lazy-fusion threshold (sweep via --theta).
    "resnet50-csc": dict(sizes=RESNET50, model="resnet50", csc=True, theta=64 << 20, sparsity=0.9),
}
CSC_SUB = "alexnet-csc"  # the `csc` sub-object of the default line


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


def numa_bind(torch, local):
    """Run this rank on the CPUs local to its GPU (sysfs local_cpulist of the GPU's PCI device),
    so the pinned host buffers of the e2e leg are first-touched on the GPU's NUMA node: a remote
    node puts every H2D/D2H byte across the socket link (measured: 3.5 vs 2.2 ms per e2e step)."""
    try:
        p = torch.cuda.get_device_properties(local)
        bus = "%04x:%02x:%02x.0" % (p.pci_domain_id, p.pci_bus_id, p.pci_device_id)
        base = f"/sys/bus/pci/devices/{bus}"
        cpus = set()
        for part in open(f"{base}/local_cpulist").read().strip().split(","):
            lo, _, hi = part.partition("-")
            cpus.update(range(int(lo), int(hi or lo) + 1))
        cpus &= os.sched_getaffinity(0)
        if not cpus:
            return None
        os.sched_setaffinity(0, cpus)
        node = int(open(f"{base}/numa_node").read().strip())
        return {"gpu_pci": bus, "numa_node": node, "cpus": len(cpus)}
    except Exception:  # noqa: BLE001 - best effort (no sysfs, no affinity rights)
        return None


def host_cpu():
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count()}


class ClockSampler:
    """SM clocks + throttle reasons while the timed work executes.

    sample_now() is called by the main thread right after the timed steps are enqueued
    (the GPU is still executing them). A separate nvidia-smi process (-lms 50) records the
    whole run for throttle reasons."""

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


def ring_bus_bytes(esz, world, window_elems):
    """NCCL busBw convention: 2(N-1)/N * K per rank (K = window bytes)."""
    if world == 1:
        return 0
    return sum(2 * (world - 1) * (wl * esz) / world for wl in window_elems)


def config_of(workload, wl, world):
    """The workload description both arms print (identical keys and values)."""
    theta = wl["theta"]
    return {"workload": workload, "gradient_set": wl["model"],
            "tensors": len(wl["sizes"]), "elements": sum(wl["sizes"]),
            "wire": "fp16", "chunk": 32000,
            "theta_bytes": "inf" if theta == THETA_INF else theta,
            "csc_sparsity": wl.get("sparsity") if wl["csc"] else None,
            "inputs": "SURVEY 8(d) mt19937_64(1234+rank+7919*step) uniform(-1,1)*2^-(id mod 7)",
            "parallelism": f"dp{world}", "global_batch": None, "seq_len": None}


# ---- reference arm ------------------------------------------------------------------------------
def reference_arm(args, workload, wl, world, rank):
    """--impl reference: the reference's own CPU implementation (oracle/_ref = the unmodified
    library compiled from /root/reference) on the host cores, ranks as threads, on the same
    seeded gradients. Rank 0 alone runs it; the others exit without work."""
    if rank != 0:
        return 0
    from oracle.oracle import Reference
    ref = Reference()
    kw = dict(chunk=32000, dtype=1, theta=wl["theta"], csc=wl["csc"], final_sparsity=wl.get("sparsity", 0.9))
    warm = max(0, args.warmup)
    # one probe step bounds the run: the timed steps fit a ~100 s budget
    t0 = time.perf_counter()
    ref.time_step(world, wl["sizes"], steps=1, warmup=0, **kw)
    per = time.perf_counter() - t0
    steps = max(1, min(args.steps, int(100.0 / max(per, 1e-3)) - warm))
    st = ref.time_step(world, wl["sizes"], steps=steps, warmup=warm, **kw)
    line = {
        "metric": "grad-sync ms/step", "value": round(st["total"], 3), "unit": "ms",
        "n_gpus": world, "steps": steps, "warmup": warm, "ms_per_step": round(st["total"], 3),
        "higher_is_better": False, "scaling": "weak", "vs_baseline": None, "dtype": "fp16",
        "data": "synthetic", "impl": "reference",
        "config": config_of(workload, wl, world),
        "stages_ms": {k: round(v, 3) for k, v in st.items()},
        "cpu_baseline": dict({"value": round(st["total"], 3), "unit": "ms", "cores": world,
                              "kind": "reference",
                              "sample": f"{steps} timed steps (median, +{warm} warm-up) of the full workload, "
                                        f"{world} rank thread(s) over InprocTransport"
                                        + (f" (steps capped from {args.steps} by a 100 s budget)"
                                           if steps < args.steps else "")},
                             **host_cpu()),
        "e2e": {"value": round(st["total"], 3), "unit": "ms", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---- our arm --------------------------------------------------------------------------------------
class Run:
    """One workload through the engine on this rank: timed steps, per-kernel marks, roofline,
    e2e, and (N=1) the step-0 parity check + CPU baseline."""

    def __init__(self, args, workload, world, rank, local, dist, allgather):
        import numpy as np
        import torch
        from paper_1902_06855_b200 import capi
        from paper_1902_06855_b200.engine import GradSync
        self.np, self.torch, self.capi = np, torch, capi
        self.args, self.workload, self.world, self.rank, self.local, self.dist = args, workload, world, rank, local, dist
        wl = dict(WORKLOADS[workload])
        if args.theta is not None and workload == args.workload:
            wl["theta"] = THETA_INF if args.theta < 0 else args.theta
        self.wl = wl
        self.sizes = wl["sizes"]
        self.csc = wl["csc"]
        self.sync = GradSync(self.sizes, rank=rank, world=world, device=local, theta=wl["theta"], csc=self.csc,
                             final_sparsity=wl.get("sparsity", 0.9), allgather=allgather,
                             dense_mode=args.dense_mode, csc_mode=args.csc_mode)
        self.L = self.sync.layout
        self.total = self.L.total
        self.dev = torch.device("cuda", local)
        self.stream = torch.cuda.current_stream()
        self.sp = self.stream.cuda_stream
        # rotating input sets (> 2x L2 in total): set t holds step t's seeded gradients
        in_bytes = self.total * 4
        self.n_sets = max(2, math.ceil(2 * L2_BYTES / in_bytes) + 1)
        self.inputs = [torch.from_numpy(capi.synth_grads(rank, t, self.sizes)).to(self.dev)
                       for t in range(self.n_sets)]
        self.in_bytes = in_bytes
        bounds = np.concatenate([[0], np.cumsum(self.sizes)])
        self.bounds = bounds
        import ctypes as C

        def table(flat):
            return (C.c_void_p * len(self.sizes))(*[flat[int(bounds[i]):int(bounds[i + 1])].data_ptr()
                                                     for i in range(len(self.sizes))])
        self.in_ptrs = [table(x) for x in self.inputs]
        self.outs = [torch.empty(self.total, device=self.dev) for _ in range(2)]
        self.out_ptrs = [table(x) for x in self.outs]
        self.parity_data = None

    def step(self, i):
        if self.csc:
            self.sync.csc_step(self.in_ptrs[i % self.n_sets], stream=self.sp)
        else:
            self.sync.dense_step(self.in_ptrs[i % self.n_sets], self.out_ptrs[i % 2], stream=self.sp)

    def barrier(self):
        if self.world > 1:
            self.dist.barrier()
        self.torch.cuda.synchronize()

    def allmax(self, x):
        if self.world == 1:
            return x
        t = self.torch.tensor([x], dtype=self.torch.float64, device=self.dev)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def read_state(self, name, dtype):
        from paper_1902_06855_b200 import cudart
        p, n = self.sync.state(name)
        out = self.np.empty(n // self.np.dtype(dtype).itemsize, dtype)
        cudart.memcpy(out.ctypes.data, p, out.nbytes)
        cudart.sync_device()
        return out

    def parity_steps(self):
        """The first steps of the run on the seeded inputs, their results kept on the host for
        the parity check against the reference (N=1: the cpu_baseline leg runs it)."""
        np = self.np
        if self.csc:  # step 0 is dense (sparse.cpp:45-51), step 1 sparse: check both sets + step 1's state
            rec = {}
            for t in range(2):
                self.step(t)
                self.torch.cuda.synchronize()
                rec[f"next_imp{t}"] = self.read_state("imp_next", np.uint8)
            for key in ("pool", "hg", "hu", "w"):
                rec[key] = self.read_state(key, np.uint16 if key == "pool" else np.float32)
            self.parity_data = rec
            return 2
        self.step(0)
        self.torch.cuda.synchronize()
        self.parity_data = {"pool": self.read_state("pool", np.uint16), "gavg": self.outs[0].cpu().numpy()}
        return 1

    def check_parity(self, ref):
        """Bit-exact comparison of the recorded steps with the reference library's own run
        on the same gradients (N=1)."""
        np = self.np
        d = self.parity_data
        from paper_1902_06855_b200 import capi
        if self.csc:
            grads = [[capi.synth_grads(0, t, self.sizes)] for t in range(2)]
            res = ref.csc_run(grads, self.sizes, 32000, dtype=1, theta=self.wl["theta"],
                              final_sparsity=self.wl.get("sparsity", 0.9),
                              keep=lambda k, t, r: k == "next_imp" or (t == 1 and k in ("pool_x", "hg", "hu", "w")))
            ok = all((d[f"next_imp{t}"] == res["next_imp"][t][0]).all() for t in range(2))
            ok &= (d["pool"] == res["pool_x"][1][0]).all()
            for k in ("hg", "hu", "w"):
                ok &= (d[k].view(np.uint32) == res[k][1][0].view(np.uint32)).all()
            what = "steps 0-1: selected sets, then pool, hg, hu, w after step 1"
        else:
            g0 = capi.synth_grads(0, 0, self.sizes)
            pools, gavg, _, _ = ref.dense_sync([g0], self.sizes, dtype=1, theta=self.wl["theta"])
            ok = bool((d["pool"] == pools[0]).all())
            off = self.L.offsets
            want = np.concatenate([gavg[0][int(o):int(o) + int(s)] for o, s in zip(off, self.sizes)])
            ok &= bool((d["gavg"].view(np.uint32) == want.view(np.uint32)).all())
            what = "step 0: pool and every tensor's g_avg"
        return bool(ok), what

    def measure(self, clocks=None, cpu_leg=True, e2e=True):
        args, torch, np, capi = self.args, self.torch, self.np, self.capi
        from paper_1902_06855_b200 import cudart
        first = self.parity_steps()
        warm = max(args.warmup, 0)
        for i in range(warm):
            self.step(first + i)
        self.barrier()
        launches0 = capi.lib().gf_kernel_launches()
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        self.barrier()
        t0.record(self.stream)
        h0 = time.perf_counter()
        base = first + warm
        for i in range(args.steps):
            self.step(base + i)
        t1.record(self.stream)
        host_enqueue_ms = (time.perf_counter() - h0) * 1e3 / max(args.steps, 1)
        if clocks is not None:
            clocks.sample_now()  # the GPU is still executing the queued timed steps here
        torch.cuda.synchronize()
        self.barrier()
        launches = capi.lib().gf_kernel_launches() - launches0
        self.sync.status()
        ms = self.allmax(t0.elapsed_time(t1) / max(args.steps, 1))

        # per-kernel durations: the same K steps again with an event before every kernel
        # (kept out of the headline pass: an event between two kernels costs ~3 us of GPU time)
        self.sync.set_marks(True)
        for i in range(args.steps):
            self.step(base + args.steps + i)
        torch.cuda.synchronize()
        seg_ms = self.sync.marks()
        self.sync.set_marks(False)
        self.barrier()
        self.sync.status()
        seg_ms = {k: self.allmax(v) for k, v in seg_ms.items()}
        kernel_timing = "events between kernels, second pass of the same K steps"
        if len(seg_ms) == 1 and launches == args.steps:
            seg_ms = {k: ms for k in seg_ms}
            kernel_timing = "one launch per step: t0/t1 events over the K timed launches"
        out = {"ms": ms, "launches": int(launches), "host_enqueue_ms_per_step": round(host_enqueue_ms, 4),
               "kernel_timing": kernel_timing}
        out.update(self.roofline(seg_ms))
        if self.world > 1:  # the whole step against NVLink: the ring's bytes over the step's time
            sb = out["ring_bus_bytes"] / (ms / 1e3) / 1e9
            out["step_bus"] = {"GBps": round(sb, 1), "frac_900": round(sb / NVLINK_GBS, 3),
                               "bytes": int(out["ring_bus_bytes"]),
                               "note": "2(N-1)/N x K (NCCL busBw convention) / whole step incl. pack and unpack"}
        if e2e and not args.no_e2e:
            out["e2e"] = self.e2e()
            if self.world == 1:
                out["e2e_api"] = self.e2e_api()
        if self.world == 1 and self.rank == 0 and cpu_leg and not args.no_cpu_baseline:
            out.update(self.cpu_leg())
        else:
            out["parity"] = None
            out["parity_detail"] = ("checked at N=1 by bench's cpu_baseline leg; the N>1 kernels by "
                                    "tests/test_gpu_colocated.py (full-size, vs oracle/_ref)")
        return out

    def roofline(self, seg_ms):
        np = self.np
        hbm_peak, peak_src = load_peaks()
        total, world, esz = self.total, self.world, 2
        from paper_1902_06855_b200.engine import dense_windows
        _, wlen = dense_windows(self.L, esz, self.wl["theta"])
        algo = {"pack": total * 6, "unpack": total * 6, "pack_correct": total * 14,
                "pack_unpack": total * 10,  # N=1: g in (4), pool out (2), g_avg out (4)
                "pack_push": total * 6,     # the routed pack: HBM 6 B/el (its NVLink stores ride on it)
                "norms": total * 2}
        if self.csc:
            staged = int(self.read_state("plan_cur", np.uint64)[0])
            algo["pack_correct"] = total * 14 + (staged * 2 if world > 1 else 0)
            # N>1: the selected chunks (g, hg in; hg, pool, staging out) and the others (g, hg in; hg, pool out)
            algo["pack_correct_sel"] = staged * 16
            algo["pack_correct_rest"] = (total - staged) * 14
            algo["scatter"] = staged * 4
            algo["sgd_update"] = staged * 18
            ring_bytes = ring_bus_bytes(esz, world, [staged])
        else:
            ring_bytes = ring_bus_bytes(esz, world, wlen)
        for k in ("ring", "ring_scatter", "ring_unpack"):
            algo[k] = ring_bytes if world > 1 else None
        # rspush splits the ring's bytes: the routed pack pushes the reduce-scatter half (its
        # binding bound at N>1: the HBM side is 6 B/el), rsp_kernel pushes the all-gather half
        if world > 1 and not self.csc:
            algo["rsp"] = ring_bytes / 2
            algo["pack_push"] = ring_bytes / 2
        nvlink = ("ring", "ring_scatter", "ring_unpack", "rsp") + (("pack_push",) if world > 1 else ())
        kernels = {}
        for k, v in seg_ms.items():
            d = {"ms": round(v, 4)}
            if algo.get(k):
                d["GBps"] = round(algo[k] / (v / 1e3) / 1e9, 1)
                if k in nvlink:
                    d["busbw_frac_900"] = round(d["GBps"] / NVLINK_GBS, 3)
                else:
                    d["frac_hbm"] = round(d["GBps"] / hbm_peak, 3)
            kernels[k] = d
        dom = max(seg_ms, key=lambda k: seg_ms[k]) if seg_ms else None
        roof = None
        if dom is not None and algo.get(dom):
            ach = algo[dom] / (seg_ms[dom] / 1e3) / 1e9
            if dom in nvlink:
                roof = {"bound": "nvlink", "achieved": round(ach, 1), "peak": NVLINK_GBS, "unit": "GB/s",
                        "frac": round(ach / NVLINK_GBS, 3), "traffic": None, "kernel": dom,
                        "peak_src": "NVLink 5 nominal 900 GB/s/direction (measured SM-driven peer copy ~660-730)"}
                if dom == "ring_unpack":
                    roof["note"] = "the unpack HBM pass sits inside the time the NVLink bus bytes are divided by"
            else:
                roof = {"bound": "hbm", "achieved": round(ach, 1), "peak": hbm_peak, "unit": "GB/s",
                        "frac": round(ach / hbm_peak, 3), "traffic": None, "kernel": dom, "peak_src": peak_src}
        if roof is not None:
            try:
                with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
                    tr = json.load(f)
                kname = {"pack": "pack_kernel", "pack_unpack": "pack_kernel", "unpack": "unpack_kernel",
                         "pack_correct": "pack_correct_kernel", "pack_correct_rest": "pack_correct_kernel",
                         "sgd_update": "csc_sgd_kernel",
                         "scatter": "compact_kernel", "select": "select_kernel", "pack_push": "pack_push_kernel",
                         "rsp": "rsp_kernel"}.get(dom)
                ent = tr.get(self.workload, {}).get(kname or "", {})
                if ent:
                    roof["traffic"] = ent["dram_bytes_per_launch"]
                    roof["traffic_note"] = "ncu --set full, cold cache, profiles/ncu_traffic.json"
            except Exception:
                pass
        bus = None
        if world > 1:
            rk = next((k for k in ("ring", "ring_unpack", "ring_scatter") if k in seg_ms), None)
            if rk:
                bus = round(ring_bytes / (seg_ms[rk] / 1e3) / 1e9, 1)
            elif "rsp" in seg_ms and "pack_push" in seg_ms:  # the two kernels that carry the ring's bytes
                bus = round(ring_bytes / ((seg_ms["rsp"] + seg_ms["pack_push"]) / 1e3) / 1e9, 1)
        return {"kernels": kernels, "roofline": roof, "bus_gbs": bus, "ring_bus_bytes": ring_bytes}

    def e2e(self):
        """The same step through the C-ABI with HOST buffers: every step the H2D of its
        gradients from pinned memory and the D2H of its result (g_avg, or the updated weights
        for CSC) are inside the timed region; double-buffered on three streams, so the H2D of
        step i+1 overlaps the D2H of step i."""
        torch = self.torch
        from paper_1902_06855_b200 import cudart
        total, csc = self.total, self.csc
        h_in = [torch.empty(total, dtype=torch.float32, pin_memory=True) for _ in range(2)]
        for i, h in enumerate(h_in):
            h.copy_(self.inputs[i].cpu())
        h_out = [torch.empty(total, dtype=torch.float32, pin_memory=True) for _ in range(2)]
        d2h = total * 4
        s_in, s_out = torch.cuda.Stream(device=self.dev), torch.cuda.Stream(device=self.dev)
        wptr = self.sync.state("w")[0] if csc else None
        stream = self.stream

        def run_e2e(k):
            ev_in = [torch.cuda.Event() for _ in range(k)]
            ev_comp = [torch.cuda.Event() for _ in range(k)]
            ev_out = [torch.cuda.Event() for _ in range(k)]
            for i in range(k):
                slot = i % 2
                if i >= 2:
                    s_in.wait_event(ev_comp[i - 2])  # step i-2 finished reading this input slot
                with torch.cuda.stream(s_in):
                    self.inputs[slot].copy_(h_in[slot], non_blocking=True)
                ev_in[i].record(s_in)
                stream.wait_event(ev_in[i])
                if i >= 1:
                    stream.wait_event(ev_out[i - 1])
                self.step(slot)
                ev_comp[i].record(stream)
                s_out.wait_event(ev_comp[i])
                if csc:  # the updated weights w (engine-owned) leave the device
                    cudart.memcpy(h_out[slot].data_ptr(), wptr, d2h, s_out.cuda_stream)
                else:
                    with torch.cuda.stream(s_out):
                        h_out[slot].copy_(self.outs[slot], non_blocking=True)
                ev_out[i].record(s_out)
            return ev_out[-1]

        run_e2e(3)
        self.torch.cuda.synchronize()
        self.barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(s_in)
        stream.wait_event(e0)
        last = run_e2e(self.args.steps)
        s_out.wait_event(last)
        e1.record(s_out)
        torch.cuda.synchronize()
        ems = self.allmax(e0.elapsed_time(e1) / max(self.args.steps, 1))
        # the staging copies above overwrote input sets 0/1 with sets 0/1: unchanged inputs
        return {"value": round(ems, 4), "unit": "ms", "h2d_bytes_per_step": total * 4,
                "d2h_bytes_per_step": d2h,
                "path": "C-ABI gf_engine_* with pinned host grads in / results out, double-buffered: "
                        "H2D of step i+1 overlaps D2H of step i"}

    def e2e_api(self):
        """The same workload through the reference-shaped C++ API (gflow::GradientPool /
        FusionEngine / SparseState, what a drop-in user of the reference calls): a train_worker
        sync loop with pinned host gradients (write_tensor per tensor) and the update read
        (read_averaged: unpack + D2H) or the CSC calls; wall clock, N=1 (gflowpy.bench_api)."""
        try:
            import paper_1902_06855_b200.gflowpy as gp
            r = gp.bench_api(self.sizes, steps=self.args.steps, warmup=max(self.args.warmup, 1),
                             theta=self.wl["theta"], csc=self.csc, final_sparsity=self.wl.get("sparsity", 0.9))
            return {"value": round(r["ms_per_step"], 4), "unit": "ms", "h2d_bytes_per_step": r["h2d_bytes_per_step"],
                    "d2h_bytes_per_step": r["d2h_bytes_per_step"],
                    "path": "gflow:: C++ API (GradientPool.write_tensor per tensor from pinned host memory, "
                            "FusionEngine windows, wait_all, read_averaged / SparseState calls), wall clock"}
        except Exception as e:  # pragma: no cover
            return {"error": str(e)[:200]}

    def cpu_leg(self):
        """N=1, rank 0: the reference library (oracle/_ref) as the checker of the recorded steps
        and as the timed CPU baseline on a bounded sample (3 steps + 1 warm-up)."""
        try:
            from oracle.oracle import Reference
            if not Reference.available():
                return {"cpu_baseline": {"error": "oracle/_ref not built"}, "parity": None}
            ref = Reference()
            ok, what = self.check_parity(ref)
            st = ref.time_step(1, self.sizes, chunk=32000, dtype=1, theta=self.wl["theta"], csc=self.csc,
                               final_sparsity=self.wl.get("sparsity", 0.9), steps=3, warmup=1)
            cpu = dict({"value": round(st["total"], 3), "unit": "ms", "cores": 1, "kind": "reference",
                        "sample": "3 timed steps (median, +1 warm-up) of the full workload, 1 rank thread, "
                                  "the same seeded gradients",
                        "stages_ms": {k: round(v, 2) for k, v in st.items()}}, **host_cpu())
            return {"cpu_baseline": cpu, "parity": ok,
                    "parity_detail": f"bit-exact vs the reference library (oracle/_ref) on the bench's own "
                                     f"seeded inputs: {what}"}
        except Exception as e:  # pragma: no cover
            return {"cpu_baseline": {"error": str(e)[:200]}, "parity": None}

    def close(self):
        self.sync.close()


def nccl_compare(run):
    torch, dist = run.torch, run.dist
    x = torch.zeros(run.total, dtype=torch.float16, device=run.dev)
    for _ in range(3):
        dist.all_reduce(x)
    run.barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(run.stream)
    for _ in range(run.args.steps):
        dist.all_reduce(x)
    e1.record(run.stream)
    torch.cuda.synchronize()
    nms = run.allmax(e0.elapsed_time(e1) / max(run.args.steps, 1))
    w = run.world
    return {"ms": round(nms, 4), "busbw_GBps": round(2 * (w - 1) / w * run.total * 2 / (nms / 1e3) / 1e9, 1)}


SELECT_PHASES = ["finalize+push", "entry_wait", "sum", "exit_wait", "topk", "plan"]


def ring_trace(run):
    """Device timestamps of CTA 0 of the NVLink kernel (diagnostic, outside the timed region)."""
    import ctypes as C
    capi = run.capi
    capi.call("gf_comm_set_trace", run.sync.comm, 1)
    rec = []
    for i in range(run.args.steps):
        run.barrier()
        run.step(i)
        run.torch.cuda.synchronize()
        t = (C.c_uint64 * 11)()
        capi.call("gf_comm_trace_n", run.sync.comm, t, 11)
        rec.append([t[1] - t[0], t[2] - t[1], t[3] - t[2]] +
                   ([t[5] - t[4], t[6] - t[5], t[7] - t[6], t[8] - t[7], t[9] - t[8], t[10] - t[9]]
                    if run.csc else []))
    capi.call("gf_comm_set_trace", run.sync.comm, 0)
    if run.world == 1:  # no NVLink kernel: the selection's phases only
        return {"select_phases_us": [round(statistics.median(r[j] for r in rec) / 1e3, 2) for j in range(3, 9)],
                "select_phase_names": SELECT_PHASES}
    med = [statistics.median(r[j] for r in rec) / 1e3 for j in range(3)]
    out = {"entry_wait_us": round(run.allmax(med[0]), 2), "body_us": round(run.allmax(med[1]), 2),
           "exit_wait_us": round(run.allmax(med[2]), 2)}
    per_rank = [None] * run.world
    run.dist.all_gather_object(per_rank, [round(m, 2) for m in med])
    out["per_rank_entry_body_exit_us"] = per_rank
    if run.csc:
        out["select_phases_us"] = [round(run.allmax(statistics.median(r[j] for r in rec) / 1e3), 2)
                                   for j in range(3, 9)]
        out["select_phase_names"] = SELECT_PHASES
    return out


def overlap_probe(run, backward_ms):
    """Dense sync overlapped with a synthetic backward (fusion.cpp:72-123)."""
    torch = run.torch
    sizes, total, sync, sp = run.sizes, run.total, run.sync, run.sp
    A = torch.randn(2048, 4096, dtype=torch.bfloat16, device=run.dev)
    B = torch.randn(4096, 4096, dtype=torch.bfloat16, device=run.dev)
    Cm = torch.empty(2048, 4096, dtype=torch.bfloat16, device=run.dev)
    for _ in range(20):
        torch.matmul(A, B, out=Cm)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(run.stream)
    for _ in range(50):
        torch.matmul(A, B, out=Cm)
    e1.record(run.stream)
    torch.cuda.synchronize()
    gemm_ms = e0.elapsed_time(e1) / 50
    n_gemm = max(1, round(backward_ms / gemm_ms))
    reps = {tid: int(round(n_gemm * sizes[tid - 1] / total)) for tid in range(1, len(sizes) + 1)}

    def backward(i, with_sync):
        if with_sync:
            sync.begin_iteration(run.in_ptrs[i % run.n_sets], run.out_ptrs[i % 2], stream=sp)
        for tid in range(len(sizes), 0, -1):
            for _ in range(reps[tid]):
                torch.matmul(A, B, out=Cm)
            if with_sync:
                sync.tensor_complete(tid)
        if with_sync:
            sync.finalize_iteration()

    for i in range(3):
        backward(i, False)
        backward(i, True)
    run.barrier()
    K = run.args.steps
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(2 * K + 1)]
    evs[0].record(run.stream)
    for i in range(K):
        backward(i, False)
        evs[2 * i + 1].record(run.stream)
        backward(i, True)
        evs[2 * i + 2].record(run.stream)
    torch.cuda.synchronize()
    run.barrier()
    t_bw = [evs[2 * i].elapsed_time(evs[2 * i + 1]) for i in range(K)]
    t_both = [evs[2 * i + 1].elapsed_time(evs[2 * i + 2]) for i in range(K)]
    bw = run.allmax(statistics.median(t_bw))
    both = run.allmax(statistics.median(t_both))
    return {"backward_ms": round(bw, 4), "backward_plus_sync_ms": round(both, 4),
            "exposed_sync_ms": round(both - bw, 4),
            "method": "backward-only and backward+sync steps alternate; medians, max over ranks",
            "backward": f"{sum(reps.values())} bf16 GEMMs 2048x4096x4096 per step, by tensor size"}


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
    ap.add_argument("--no-csc", action="store_true", help="skip the csc sub-object")
    ap.add_argument("--trace", action="store_true", help="report NVLink kernel CTA-0 timestamps (diagnostic)")
    ap.add_argument("--overlap", type=float, default=0.0, metavar="BACKWARD_MS",
                    help="also measure the dense sync overlapped with a synthetic backward of this many ms")
    ap.add_argument("--dense-mode", default="auto", choices=["auto", "pull", "push", "rspush"],
                    help="dense N>1: rspush (pack pushes the reduce-scatter operands to their owners, "
                         "local reduce + all-gather push, unpack), pull (pack + pull RS/AG fused with "
                         "unpack), push (pack + push-pull ring + unpack); auto = rspush")
    ap.add_argument("--csc-mode", default="auto", choices=["auto", "pull", "push"],
                    help="CSC N>1 exchange: pull (selected chunks routed to their owners by the pack, "
                         "local RS + pull AG straight into the pool) or push (push-pull ring + fused "
                         "write-back); auto = pull from 4 ranks, else push")
    args = ap.parse_args()

    world = env_int("WORLD_SIZE", 1)
    rank = env_int("RANK", 0)
    local = env_int("LOCAL_RANK", 0)
    wl = dict(WORKLOADS[args.workload])
    if args.theta is not None:
        wl["theta"] = THETA_INF if args.theta < 0 else args.theta
    if args.impl == "reference":
        return reference_arm(args, args.workload, wl, world, rank)

    import torch
    import torch.distributed as dist

    from paper_1902_06855_b200 import cudart

    torch.cuda.set_device(local)
    cudart.set_device(local)  # the library's CUDA runtime (may differ from torch's) on the same GPU
    numa = None if os.environ.get("GF_BENCH_NO_NUMA") else numa_bind(torch, local)  # before any pinned buffer
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    def allgather(b):
        out = [None] * world
        dist.all_gather_object(out, b)
        return out

    clocks = ClockSampler(local)
    run = Run(args, args.workload, world, rank, local, dist, allgather)
    res = run.measure(clocks=clocks)
    extra = {}
    if args.trace and (world > 1 or run.csc):
        extra["ring_trace"] = ring_trace(run)
    if args.overlap > 0 and not run.csc:
        extra["overlap"] = dict(overlap_probe(run, args.overlap), sync_alone_ms=round(res["ms"], 4))
    nccl = nccl_compare(run) if world > 1 else None
    exchange = "none (N=1)" if world == 1 else (run.sync.csc_mode if run.csc else run.sync.dense_mode)
    run.close()

    csc_sub = None
    if not args.no_csc and not run.csc:
        crun = Run(args, CSC_SUB, world, rank, local, dist, allgather)
        c = crun.measure(e2e=False)
        sel = c["kernels"].get("select", {}).get("ms")
        csc_sub = {"workload": CSC_SUB, "config": config_of(CSC_SUB, crun.wl, world), "value": round(c["ms"], 4),
                   "unit": "ms", "kernels": c["kernels"], "roofline": c["roofline"], "bus_gbs": c["bus_gbs"],
                   "select_us": round(sel * 1e3, 2) if sel else None, "gpu_launches": c["launches"],
                   "exchange": "none (N=1)" if world == 1 else crun.sync.csc_mode,
                   "parity": c["parity"], "parity_detail": c.get("parity_detail"),
                   "cpu_baseline": c.get("cpu_baseline")}
        crun.close()
    clk = clocks.stop()

    if rank == 0:
        line = {
            "metric": "grad-sync ms/step", "value": round(res["ms"], 4), "unit": "ms", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(res["ms"], 4),
            "higher_is_better": False, "scaling": "weak", "vs_baseline": None, "dtype": "fp16",
            "data": "synthetic", "config": config_of(args.workload, wl, world),
            "exchange": exchange,
            "l2_policy": f"{run.n_sets} rotating input sets of {run.in_bytes >> 20} MiB (> 126 MB L2 in total)",
            "parity": res["parity"], "parity_detail": res.get("parity_detail"),
            "bus_gbs": res["bus_gbs"], "step_bus": res.get("step_bus"), "kernels": res["kernels"],
            "kernel_timing": res["kernel_timing"],
            "roofline": res["roofline"], "cpu_baseline": res.get("cpu_baseline"), "e2e": res.get("e2e"),
            "e2e_api": res.get("e2e_api"),
            "nccl_allreduce": nccl, "gpu_launches": res["launches"], "clocks": clk,
            "host_enqueue_ms_per_step": res["host_enqueue_ms_per_step"], "csc": csc_sub, "host_numa": numa,
        }
        line.update(extra)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())

# SPDX-License-Identifier: Apache-2.0
"""Render a scripts/sweep_bw.py log as profiles/sweep_bw_<tag>.md + .jsonl. Usage: sweep_md.py LOG TAG"""
import json
import sys

log, tag = sys.argv[1], sys.argv[2]
rows = [json.loads(x) for x in open(log) if x.startswith("{")]
n = rows[0]["n_gpus"]


def fmt(b):
    for u, s in ((1 << 30, "GiB"), (1 << 20, "MiB"), (1 << 10, "KiB")):
        if b >= u:
            return f"{b // u} {s}"
    return str(b)


out = [f"# Allreduce bandwidth sweep, {n} x B200 (SURVEY §8(d) config 5), {tag}", "",
       f"`torchrun --nproc-per-node {n} scripts/sweep_bw.py`: device time per call (CUDA events on the launching "
       "stream, max over ranks), fp16, busBW = 2(N-1)/N x bytes / t in GB/s per GPU per direction "
       "(NVLink 5 nominal 900).", "",
       "| bytes | ring (push-pull) µs | busBW | pull RS/AG + fp32 unpack µs | busBW | CSC exchange (10 % of "
       "chunks) µs | staged bytes | busBW | NCCL all_reduce µs | busBW |",
       "|---|---|---|---|---|---|---|---|---|---|"]
for r in rows:
    out.append(f"| {fmt(r['bytes'])} | {r['ring_us']} | {r['ring_busbw']} | {r['pull_unpack_us']} | "
               f"{r['pull_unpack_busbw']} | {r.get('csc_us')} | {r.get('csc_staged_bytes')} | {r.get('csc_busbw')} | "
               f"{r['nccl_us']} | {r['nccl_busbw']} |")
out += ["", f"Raw JSON lines: `sweep_bw_{tag}_n{n}.jsonl`."]
open(f"profiles/sweep_bw_{tag}_n{n}.md", "w").write("\n".join(out) + "\n")
open(f"profiles/sweep_bw_{tag}_n{n}.jsonl", "w").write("".join(json.dumps(r) + "\n" for r in rows))

# SPDX-License-Identifier: Apache-2.0
"""Summarise ncu evidence into profiles/: per-kernel launch shares (from a
--metrics gpu__time_duration.sum launch list) and key counters of a --set full report.

    python scripts/ncu_summary.py launches.csv [prof.ncu-rep] > profiles/<name>.md
"""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_pct_of_peak"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram_throughput_pct"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_pct"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_active_pct"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps_active_pct"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("lts__t_bytes.sum", "l2_bytes"),
]


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = defaultdict(list)
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                v = float(d["Metric Value"].replace(",", ""))
                if d.get("Metric Unit") == "us":
                    v *= 1000.0
                elif d.get("Metric Unit") == "ms":
                    v *= 1e6
                agg[d["Kernel Name"].split("(")[0]].append(v)
    return agg


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return []
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")].split("(")[0]}
        for k, name in KEYS:
            if k in hdr:
                d[name] = f"{r[hdr.index(k)]} {units[hdr.index(k)]}".strip()
        res.append(d)
    return res


def main():
    lp = sys.argv[1]
    agg = launches(lp)
    tot = sum(sum(v) for v in agg.values())
    print(f"# ncu launch list: `{lp.split('/')[-1]}`\n")
    print("Cold-cache, serialised per-launch times (`--metrics gpu__time_duration.sum "
          "--clock-control none`); compare SHARES with bench.py, not absolutes.\n")
    print("| kernel | launches | mean µs | share of all launch time |")
    print("|---|---|---|---|")
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        print(f"| `{k}` | {len(v)} | {sum(v) / len(v) / 1e3:.2f} | {100 * sum(v) / tot:.1f} % |")
    if len(sys.argv) > 2:
        print(f"\n# ncu --set full: `{sys.argv[2].split('/')[-1]}`\n")
        seen = set()
        for d in full(sys.argv[2]):
            if d["kernel"] in seen:
                continue
            seen.add(d["kernel"])
            print(f"## `{d['kernel']}`\n")
            print("```\n" + json.dumps(d, indent=1) + "\n```\n")


if __name__ == "__main__":
    main()

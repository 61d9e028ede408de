# SPDX-License-Identifier: Apache-2.0
"""profiles/ncu_traffic.json from `ncu --set full` reports: DRAM bytes (read + write) per
launch of each kernel, the `traffic` field of bench.py's roofline.

    python scripts/ncu_traffic.py TAG workload=path.ncu-rep [workload=path.ncu-rep ...]
"""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict


def per_launch(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                          "dram__bytes_read.sum,dram__bytes_write.sum"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    agg = defaultdict(list)
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")].replace("void ", "").replace("<unnamed>::", "")
        name = name.split("(")[0].split("<")[0]
        b = 0.0
        for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            i = hdr.index(m)
            b += float(r[i].replace(",", "")) * mult.get(units[i], 1)
        agg[name].append(b)
    return {k: {"dram_bytes_per_launch": int(sum(v) / len(v)), "launches_captured": len(v)} for k, v in agg.items()}


def main():
    tag = sys.argv[1]
    res = {}
    for arg in sys.argv[2:]:
        w, rep = arg.split("=", 1)
        res[w] = per_launch(rep)
    res["_source"] = (f"ncu --set full --clock-control none (scripts/profile_n1.sh {tag}), "
                      "dram__bytes_read.sum + dram__bytes_write.sum per launch, cold cache")
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()

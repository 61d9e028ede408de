# SPDX-License-Identifier: Apache-2.0
"""Markdown table of ncu NVLink/DRAM counters per kernel from scripts/diag/ncu_nvl.sh CSVs.
usage: python scripts/nvl_summary.py LABEL:file.csv [LABEL:file.csv ...]"""
import collections
import csv
import sys


def rows_of(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    if not rows:
        return []
    h = rows[0]
    ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    d = collections.OrderedDict()
    for r in rows[1:]:
        name = r[ki].split("(")[0].replace("void <unnamed>::", "").replace("<unnamed>::", "")
        d.setdefault((r[ii], name), {})[r[mi]] = float(r[vi].replace(",", ""))
    agg = collections.OrderedDict()  # kernel -> list of launches
    for (_, name), v in d.items():
        agg.setdefault(name, []).append(v)
    return agg


def main():
    print("| config | kernel | launches | us/launch | NVLink TX user MB | TX raw MB | RX user MB | RX raw MB |"
          " user GB/s (max TX,RX) | raw GB/s | DRAM read MB | DRAM write MB |")
    print("|---|---|---|---|---|---|---|---|---|---|---|---|")
    for arg in sys.argv[1:]:
        label, path = arg.split(":", 1)
        for name, ls in rows_of(path).items():
            m = lambda k: sum(x.get(k, 0.0) for x in ls) / len(ls)  # noqa: E731
            t = m("gpu__time_duration.sum") / 1e3
            tu, tr = m("nvltx__bytes_data_user.sum"), m("nvltx__bytes.sum")
            ru, rr = m("nvlrx__bytes_data_user.sum"), m("nvlrx__bytes.sum")
            print(f"| {label} | `{name}` | {len(ls)} | {t:.1f} | {tu / 1e6:.1f} | {tr / 1e6:.1f} | {ru / 1e6:.1f} | "
                  f"{rr / 1e6:.1f} | {max(tu, ru) / t / 1e3:.0f} | {max(tr, rr) / t / 1e3:.0f} | "
                  f"{m('dram__bytes_read.sum') / 1e6:.1f} | {m('dram__bytes_write.sum') / 1e6:.1f} |")


if __name__ == "__main__":
    main()

"""Per-kernel time share, DRAM bytes and achieved HBM bandwidth from an ncu launch list
(--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv),
as a markdown table; the HBM peak is MEASURED_PEAKS.json's copy bandwidth.

    python tools/kernel_table.py LIST.csv [top]
"""
import collections
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main(path, top=24):
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, mi, vi, ui, ii = (h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"),
                          h.index("Metric Unit"), h.index("ID"))
    scale = {"ns": 1e-9, "us": 1e-6, "ms": 1e-3, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0, "byte": 1.0, "Kbyte": 1e3,
             "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
    per = collections.defaultdict(dict)
    names = {}
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
        per[r[ii]][r[mi]] = v
        names[r[ii]] = r[ki].split("(")[0].replace("void ", "")[:64]
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for i, m in per.items():
        a = agg[names[i]]
        a[0] += 1
        a[1] += m.get("gpu__time_duration.sum", 0.0)
        a[2] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
    tot = sum(a[1] for a in agg.values())
    print("| kernel | launches | time (ms) | share | DRAM bytes (GB) | achieved GB/s | of peak |")
    print("| --- | --- | --- | --- | --- | --- | --- |")
    for k, (n, t, b) in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        gbs = b / t / 1e9 if t > 0 else 0.0
        print(f"| `{k}` | {n} | {t * 1e3:.2f} | {100 * t / tot:.1f}% | {b / 1e9:.2f} | {gbs:.0f} | {gbs / peak:.2f} |")
    print(f"| total | {sum(a[0] for a in agg.values())} | {tot * 1e3:.2f} | | | | |")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 24)

"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list by kernel."""
import collections
import csv
import sys


def main(path, top=25):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[hi + 1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        name = r[ki].split("(")[0].replace("void ", "")[:58]
        v = float(r[vi].replace(",", ""))
        v *= {"usecond": 1e3, "msecond": 1e6, "second": 1e9}.get(r[ui], 1.0)
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(v[1] for v in agg.values())
    print(f"{'kernel':58s} {'launches':>8s} {'ms':>9s} {'share':>6s}")
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        print(f"{k:58s} {v[0]:8d} {v[1] / 1e6:9.2f} {100 * v[1] / tot:5.1f}%")
    print(f"{'total':58s} {sum(v[0] for v in agg.values()):8d} {tot / 1e6:9.2f}")


if __name__ == "__main__":
    main(sys.argv[1])

"""Hottest SASS instructions (by warp-stall samples and executed instructions) of one
kernel in an ncu report: python tools/ncu_sass_hot.py REPORT KERNEL_REGEX [N]."""
import collections
import csv
import subprocess
import sys


def main(path, kernel, top=30):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "-k", f"regex:{kernel}", "--launch-count", "1"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hi = [i for i, r in enumerate(rows) if "Source" in r and "Instructions Executed" in r][0]
    hdr = rows[hi]
    si, ii = hdr.index("Source"), hdr.index("Instructions Executed")
    st = hdr.index("Warp Stall Sampling (All Samples)")
    seen, data = set(), []
    for r in rows[hi + 1:]:
        if len(r) <= ii or r[0] in seen:
            continue
        seen.add(r[0])
        try:
            data.append((r[0], r[si].strip(), float(r[ii] or 0), float(r[st] or 0)))
        except ValueError:
            pass
    ti = sum(d[2] for d in data) or 1
    ts = sum(d[3] for d in data) or 1
    print(f"instructions {ti:.3e}, stall samples {ts:.0f}")
    ops = collections.defaultdict(lambda: [0.0, 0.0])
    for _, s, v, w in data:
        op = s.split()[1] if s.startswith("@") else (s.split() or ["?"])[0]
        ops[op.split(".")[0]][0] += v
        ops[op.split(".")[0]][1] += w
    for k, (v, w) in sorted(ops.items(), key=lambda x: -x[1][0])[:12]:
        print(f"  {k:10s} {100 * v / ti:5.1f}% instr {100 * w / ts:5.1f}% stall")
    print("hottest by stall:")
    for a, s, v, w in sorted(data, key=lambda x: -x[3])[:top]:
        print(f"  {a[-5:]} {100 * w / ts:5.1f}% st {100 * v / ti:5.2f}% in  {s[:70]}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 30)

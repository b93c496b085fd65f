"""Per-kernel totals of the LAST step in an ncu launch-list CSV (gpu__time_duration.sum and,
when captured, dram bytes). Usage: python tools/launch_table.py <launches.csv> [first-kernel-of-step]"""
import collections
import csv
import sys


def main(path, first=None):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h, data = rows[hi], rows[hi + 1:]
    ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    per, names = collections.defaultdict(dict), {}
    for r in data:
        per[r[ii]][r[mi]] = float(r[vi].replace(",", ""))
        names[r[ii]] = r[ki].split("(")[0]
    ids = sorted(per, key=int)
    start = ids[0]
    if first:
        starts = [i for i in ids if first in names[i]]
        start = starts[-1]
    agg = collections.OrderedDict()
    for i in ids:
        if int(i) < int(start):
            continue
        d = per[i]
        a = agg.setdefault(names[i], [0, 0.0, 0.0, 0.0])
        a[0] += 1
        a[1] += d.get("gpu__time_duration.sum", 0)
        a[2] += d.get("dram__bytes_read.sum", 0)
        a[3] += d.get("dram__bytes_write.sum", 0)
    tot = sum(a[1] for a in agg.values())
    for n, a in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{n[:56]:56s} {a[0]:4d} {a[1] / 1e3:10.1f} us {100 * a[1] / tot:5.1f}% {a[2] / 1e9:8.3f} GB rd {a[3] / 1e9:7.3f} GB wr")
    print(f"total {tot / 1e6:.3f} ms")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None)

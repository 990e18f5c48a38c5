"""Per-kernel share of the launch list written by
`ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file X python bench.py ...`."""
import collections
import csv
import sys


def main(path):
    rows = [r for r in csv.reader(l for l in open(path) if l.startswith('"'))]
    h = rows[0]
    ki, vi, mi = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name")
    tot = collections.Counter()
    cnt = collections.Counter()
    for r in rows[1:]:
        if r[mi] != "gpu__time_duration.sum":
            continue
        name = r[ki].split("(")[0].split("::")[-1].split("<")[0]
        tot[name] += float(r[vi].replace(",", ""))
        cnt[name] += 1
    s = sum(tot.values())
    print("kernel, launches, mean_us, share  (ncu gpu__time_duration.sum --clock-control none; cold-cache serialised)")
    for k, v in tot.most_common():
        print(f"{k}, {cnt[k]}, {v / cnt[k] / 1e3:.1f}, {v / s:.4f}")


if __name__ == "__main__":
    main(sys.argv[1])

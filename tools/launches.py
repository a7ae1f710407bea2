"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list: time share per kernel."""
import collections
import csv
import re
import sys


def main(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    scale = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0}
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for r in rows[hdr + 1:]:
        if len(r) <= vi:
            continue
        name = re.sub(r"\(anonymous namespace\)::|<unnamed>::|void ", "", r[ki])
        name = re.sub(r"\(.*$", "", name)
        tot[name] += float(r[vi].replace(",", "")) * scale.get(r[ui], 1e-6)
        cnt[name] += 1
    T = sum(tot.values())
    print(f"{'ms':>10} {'share':>6} {'launches':>8}  kernel")
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        print(f"{v:10.2f} {100 * v / T:5.1f}% {cnt[k]:8d}  {k}")
    print(f"{T:10.2f} total ms, {sum(cnt.values())} launches")


if __name__ == "__main__":
    main(sys.argv[1])

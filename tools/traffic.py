"""Per-launch DRAM traffic of the dominant kernel from an ncu metrics CSV
(ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:K --csv).
usage: python tools/traffic.py launches.csv CONFIG OUT.json"""
import csv
import json
import sys


def main(path, k, out):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Metric Name" in r)
    h = rows[hdr]
    ni, vi, ui, ki = h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit"), h.index("Kernel Name")
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3,
             "ns": 1e-9, "us": 1e-6, "ms": 1e-3}
    tot = {"dram__bytes_read.sum": 0.0, "dram__bytes_write.sum": 0.0, "gpu__time_duration.sum": 0.0}
    ids = set()
    name = None
    for r in rows[hdr + 1:]:
        if len(r) <= vi or r[ni] not in tot:
            continue
        tot[r[ni]] += float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
        ids.add(r[0])
        name = r[ki]
    n = len(ids)
    d = {"kernel": (name or "")[:80], "launches": n, "config": int(k),
         "dram_read_bytes_per_launch": tot["dram__bytes_read.sum"] / n,
         "dram_write_bytes_per_launch": tot["dram__bytes_write.sum"] / n,
         "dram_bytes_per_launch": (tot["dram__bytes_read.sum"] + tot["dram__bytes_write.sum"]) / n,
         "ncu_ms_per_launch": 1e3 * tot["gpu__time_duration.sum"] / n,
         "source": f"ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum over all {n} launches of one cfg{k} step "
                   f"(tools/profile_step.py), averaged per launch"}
    json.dump(d, open(out, "w"), indent=1)
    print(json.dumps(d))


if __name__ == "__main__":
    main(*sys.argv[1:4])

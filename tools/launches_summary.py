"""Summarise an ncu --csv launch list (gpu__time_duration.sum [+ dram__bytes_read.sum]) per kernel/grid."""
import collections
import csv
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, mi, vi, ui, idi, gi = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit",
                                                     "ID", "Grid Size"))
    launch = {}
    for r in rows[hdr + 1:]:
        if len(r) <= vi:
            continue
        d = launch.setdefault(int(r[idi]), {"name": r[ki].split("(")[0], "grid": r[gi], "MB": 0.0})
        v = float(r[vi].replace(",", ""))
        if r[mi] == "gpu__time_duration.sum":
            d["us"] = v * {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3}.get(r[ui], 1e-3)
        elif r[mi].startswith("dram__bytes"):  # read + write
            d["MB"] += v * {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}.get(r[ui], 1.0)
    return [launch[k] for k in sorted(launch)]


def summary(path):
    seq = load(path)
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for d in seq:
        key = d["name"] + (" " + d["grid"] if "gemm" in d["name"] else "")
        a = agg[key]
        a[0] += 1
        a[1] += d["us"]
        a[2] += d["MB"]
    tot = sum(a[1] for a in agg.values())
    lines = []
    for k, (n, t, mb) in sorted(agg.items(), key=lambda x: -x[1][1]):
        gbs = mb / t * 1e3 if t else 0.0
        lines.append(f"{k[:52]:52s} n={n:5d} avg={t / n:8.2f} us  MB/launch={mb / n:8.2f}  GB/s={gbs:6.0f}  "
                     f"{100 * t / tot:5.1f}%")
    lines.append(f"total {tot / 1000:.3f} ms over {len(seq)} launches (ncu: serialised, warm L2)")
    return "\n".join(lines), seq


if __name__ == "__main__":
    print(summary(sys.argv[1])[0])

"""Summarise an ncu --csv launch list (gpu__time_duration.sum) per kernel."""
import collections
import csv
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    out = []
    for r in rows[hdr + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", ""))
        scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(r[ui], 1e-3)
        out.append((r[ki].split("(")[0], v * scale))
    return out


def summary(path):
    seq = load(path)
    agg = collections.defaultdict(lambda: [0, 0.0])
    for n, us in seq:
        agg[n][0] += 1
        agg[n][1] += us
    tot = sum(a[1] for a in agg.values())
    lines = []
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"{k[:48]:48s} n={n:4d} total={t / 1000:8.3f} ms avg={t / n:8.2f} us {100 * t / tot:5.1f}%")
    lines.append(f"total {tot / 1000:.3f} ms over {len(seq)} launches")
    return "\n".join(lines), seq


if __name__ == "__main__":
    s, seq = summary(sys.argv[1])
    print(s)
    if len(sys.argv) > 2:
        for n, us in seq[: int(sys.argv[2])]:
            print(f"  {n[:40]:40s} {us:9.2f} us")

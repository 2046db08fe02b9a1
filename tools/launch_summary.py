"""Aggregate an ncu --metrics gpu__time_duration.sum CSV launch list by kernel name."""
import collections
import csv
import re
import sys


def summarize(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[hdr + 1:]:
        if len(r) <= vi:
            continue
        m = re.search(r"([A-Za-z_0-9]+)(<[^(]*>)?\(", r[ki])
        name = (m.group(1) + (m.group(2) or "")) if m else r[ki][:40]
        v = float(r[vi].replace(",", ""))
        v *= {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(r[ui], 1e-3)
        agg[name][0] += 1
        agg[name][1] += v
    return agg


if __name__ == "__main__":
    agg = summarize(sys.argv[1])
    tot = sum(v[1] for v in agg.values())
    print("launches %d, serialized device time %.2f ms" % (sum(v[0] for v in agg.values()), tot / 1e3))
    print("| kernel | launches | total ms | avg us | share |")
    print("|---|---|---|---|---|")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print("| %s | %d | %.3f | %.1f | %.1f%% |" % (k, v[0], v[1] / 1e3, v[1] / v[0], 100 * v[1] / tot))

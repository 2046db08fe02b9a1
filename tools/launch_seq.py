"""The launches of ONE timed step in issue order, from an ncu launch list taken with
--metrics gpu__time_duration.sum,launch__grid_size,launch__block_size (bench.py --steps 1 --warmup 3).
Prints one line per launch (index, us, CTAs, running total, kernel).
Usage: python tools/launch_seq.py launches.csv [--summary]"""
import collections
import csv
import sys


def load(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    ix = {k: i for i, k in enumerate(h)}
    by = collections.OrderedDict()
    for r in rows[1:]:
        key = r[ix["ID"]]
        d = by.setdefault(key, {"k": r[ix["Kernel Name"]].split("(")[0].replace("void <unnamed>::", "").replace("<unnamed>::", "")})
        v = r[ix["Metric Value"]].replace(",", "")
        try:
            d[r[ix["Metric Name"]]] = float(v)
        except ValueError:
            d[r[ix["Metric Name"]]] = v
    return list(by.values())


def main(path, summary=False):
    ks = load(path)
    pos = [i for i, d in enumerate(ks) if "diag_mac" in d["k"]]
    starts = [p for i, p in enumerate(pos) if i == 0 or p - pos[i - 1] > 150]
    # whole file when it holds only the timed region (ENCF_NCU_REGION=1 + --profile-from-start off)
    step = ks if "--all" in sys.argv or len(starts) < 2 else ks[starts[-2]:starts[-1]]
    tot = 0.0
    for i, d in enumerate(step):
        t = d["gpu__time_duration.sum"] / 1e3
        tot += t
        g = int(d.get("launch__grid_size", 0))
        if not summary:
            print("%4d %9.1f us %7d CTAs  %8.1f ms  %s" % (i, t, g, tot / 1e3, d["k"][:70]))
    print("step: %d launches, %.2f ms serialised" % (len(step), tot / 1e3))


if __name__ == "__main__":
    main(sys.argv[1], "--summary" in sys.argv)

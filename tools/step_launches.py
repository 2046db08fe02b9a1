"""One timed step of an ncu --metrics gpu__time_duration.sum launch list (bench.py --steps 1 --warmup 3) as a
markdown table: the whole file (a capture of the timed region) or, with --split, the launches between the last two QKV
plaintext-MAC launch groups.
Usage: python tools/step_launches.py launches.csv"""
import collections
import csv
import sys


def main(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    idx = {k: i for i, k in enumerate(h)}
    ks = [(r[idx["Kernel Name"]].split("(")[0].replace("void <unnamed>::", "").replace("<unnamed>::", ""),
           float(r[idx["Metric Value"]])) for r in rows[1:] if r[idx["Metric Name"]] == "gpu__time_duration.sum"]
    pos = [i for i, (k, _) in enumerate(ks) if "diag_mac" in k]
    starts = [p for i, p in enumerate(pos) if i == 0 or p - pos[i - 1] > 150]
    # a capture of the timed region only (ENCF_NCU_REGION=1 + --profile-from-start off, one step) is the step itself
    step = ks[starts[-2]:starts[-1]] if len(starts) >= 2 and "--split" in sys.argv else ks
    agg = collections.defaultdict(lambda: [0, 0.0])
    for k, t in step:
        agg[k][0] += 1
        agg[k][1] += t / 1e3
    tot = sum(v[1] for v in agg.values())
    print("launches %d, serialized device time %.2f ms (ncu, --clock-control none, one kernel at a time)" % (len(step), tot / 1e3))
    print()
    print("| kernel | launches | total ms | avg us | share |")
    print("|---|---|---|---|---|")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print("| %s | %d | %.3f | %.1f | %.1f%% |" % (k, v[0], v[1] / 1e3, v[1] / v[0], 100 * v[1] / tot))


if __name__ == "__main__":
    main(sys.argv[1])

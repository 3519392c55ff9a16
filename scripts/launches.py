"""Summarise an ncu --metrics gpu__time_duration.sum launch list (csv)."""
import collections
import csv
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    hdr = rows[hi]
    seq = []
    for r in rows[hi + 1:]:
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = d["Kernel Name"].split("(")[0].split("<")[0].replace("void ", "").replace("sqb::", "").strip()
        v = float(d["Metric Value"].replace(",", ""))
        unit = d["Metric Unit"]
        us = v / 1e3 if unit in ("ns", "nsecond") else (v if unit in ("us", "usecond") else v * 1e3)
        seq.append((name, us))
    return seq


if __name__ == "__main__":
    seq = load(sys.argv[1])
    agg = collections.defaultdict(lambda: [0, 0.0])
    for n, v in seq:
        agg[n][0] += 1
        agg[n][1] += v
    tot = sum(v for _, v in agg.values())
    print(f"{'kernel':28s} {'launches':>8s} {'total ms':>9s} {'share':>6s} {'avg us':>8s}")
    for k, (n, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k:28s} {n:8d} {v / 1e3:9.3f} {v / tot * 100:5.1f}% {v / n:8.2f}")
    print(f"{'total':28s} {len(seq):8d} {tot / 1e3:9.3f}")
    for name in sys.argv[2:]:
        xs = [v for n, v in seq if n == name]
        idx = [i for i in (0, 1, 2, 4, 8, 16, 32, 64, 100, len(xs) - 1) if i < len(xs)]
        print(name, {i: round(xs[i], 1) for i in idx})

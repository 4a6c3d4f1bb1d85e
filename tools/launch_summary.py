"""Summarise an ncu --csv launch list (gpu__time_duration.sum) per kernel."""
import collections
import csv
import sys


def main(path, skip=0):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d["Metric Name"] == "gpu__time_duration.sum":
                data.append(d)
    data = data[skip:]
    agg = collections.defaultdict(lambda: [0, 0.0])
    for d in data:
        k = d["Kernel Name"].split("(")[0]
        k = k.replace("orth::<unnamed>::", "")[:70]
        v = float(d["Metric Value"]) * (1e-3 if d["Metric Unit"] == "ns" else 1.0)
        agg[k][0] += 1
        agg[k][1] += v
    tot = sum(v[1] for v in agg.values())
    print(f"{'kernel':70s} {'n':>5s} {'total_us':>10s} {'avg_us':>9s} {'share':>6s}")
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k:70s} {v[0]:5d} {v[1]:10.1f} {v[1] / v[0]:9.2f} {100 * v[1] / tot:5.1f}%")
    print(f"total {tot:.1f} us over {len(data)} launches")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 0)

"""Summarise an ncu --csv launch list (gpu__time_duration.sum) per kernel."""
import collections
import csv
import sys


def load(path):
    rows, hdr = [], None
    for r in csv.reader(open(path)):
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d["Metric Name"] == "gpu__time_duration.sum":
                rows.append(d)
    return rows


def main(path, steps=1):
    rows = load(path)
    agg = collections.defaultdict(lambda: [0, 0.0])
    for d in rows:
        k = d["Kernel Name"].split("(")[0][:60] + " " + d["Grid Size"]
        agg[k][0] += 1
        agg[k][1] += float(d["Metric Value"]) / 1e3
    tot = sum(v[1] for v in agg.values())
    print(f"{'us/step':>9} {'launches':>8} {'share':>6}  kernel grid")
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{v[1] / steps:9.1f} {v[0] // steps:8d} {100 * v[1] / tot:5.1f}%  {k}")
    print(f"total {tot / steps:.1f} us/step over {len(rows) // steps} launches/step")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 1)

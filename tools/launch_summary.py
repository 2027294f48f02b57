"""Per-kernel totals of an ncu launch list (--metrics gpu__time_duration.sum --csv).
python tools/launch_summary.py launches.csv"""
import collections
import csv
import sys


def main(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    ix = {h: j for j, h in enumerate(hdr)}
    agg = collections.OrderedDict()
    scale = {"ms": 1e3, "us": 1.0, "usecond": 1.0, "ns": 1e-3, "nsecond": 1e-3, "s": 1e6,
             "msecond": 1e3}
    for r in rows[start + 1:]:
        if len(r) < len(hdr) or r[ix["Metric Name"]] != "gpu__time_duration.sum":
            continue
        v = float(r[ix["Metric Value"]].replace(",", "")) * scale.get(r[ix["Metric Unit"]], 1.0)
        a = agg.setdefault(r[ix["Kernel Name"]][:90], [0, 0.0])
        a[0] += 1
        a[1] += v
    tot = sum(v[1] for v in agg.values())
    print(f"{'launches':>8} {'total ms':>10} {'share':>7}  kernel")
    for k, (c, us) in sorted(agg.items(), key=lambda x: -x[1][1])[:20]:
        print(f"{c:8d} {us / 1e3:10.2f} {us / tot * 100:6.2f}%  {k}")
    print(f"{sum(v[0] for v in agg.values())} launches, {tot / 1e3:.1f} ms total")


if __name__ == "__main__":
    main(sys.argv[1])

"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel.

python tools/ncu_summary.py gpurun_out/launches.csv [top]
"""
import collections
import csv
import sys


def main(path, top=30):
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    r = csv.reader(lines)
    hdr = next(r)
    agg = collections.defaultdict(lambda: [0, 0.0])
    scale = {"nsecond": 1.0, "usecond": 1e3, "msecond": 1e6, "second": 1e9}
    for row in r:
        d = dict(zip(hdr, row))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        k = d["Kernel Name"].split("(")[0][:70]
        v = float(d["Metric Value"].replace(",", "")) * scale.get(d["Metric Unit"], 1.0)
        agg[k][0] += 1
        agg[k][1] += v
    tot = sum(v[1] for v in agg.values())
    n = sum(v[0] for v in agg.values())
    print(f"{n} launches, {tot / 1e6:.2f} ms summed kernel time (ncu: serialised, cold caches)")
    print(f"| kernel | launches | ms | share | us/launch |\n|---|---|---|---|---|")
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        print(f"| `{k}` | {v[0]} | {v[1] / 1e6:.2f} | {100 * v[1] / tot:.1f}% | {v[1] / v[0] / 1e3:.1f} |")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)

"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv):
per-kernel total device time, share, launches, mean per launch.

python tools/launch_summary.py launches.csv [first_id]
"""
import collections
import csv
import re
import sys


def name_of(raw):
    n = raw.replace("void ", "").replace("<unnamed>::", "").replace("(anonymous namespace)::", "")
    m = re.match(r"[A-Za-z_0-9:]+(<[^()]*>)?", n)
    return m.group(0) if m else n


def main():
    path = sys.argv[1]
    first = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr = rows[hi]
    ik, iv, im, iid = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name"), hdr.index("ID")
    tot, cnt = collections.Counter(), collections.Counter()
    for r in rows[hi + 1:]:
        if len(r) <= iv or r[im] != "gpu__time_duration.sum" or int(r[iid]) < first:
            continue
        k = name_of(r[ik])
        tot[k] += float(r[iv].replace(",", ""))
        cnt[k] += 1
    T = sum(tot.values())
    print(f"total {T / 1e6:.1f} ms over {sum(cnt.values())} launches (ids >= {first})")
    print(f"{'kernel':60s} {'ms':>10s} {'share':>6s} {'n':>7s} {'us/launch':>10s}")
    for k, v in tot.most_common(25):
        print(f"{k[:60]:60s} {v / 1e6:10.1f} {100 * v / T:5.1f}% {cnt[k]:7d} {v / cnt[k] / 1e3:10.1f}")


if __name__ == "__main__":
    main()

"""Summarise any ncu --metrics gpu__time_duration.sum --csv launch list:
launch count and summed device time per kernel."""
import csv
import sys
from collections import defaultdict


def main(path, top=15):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h, d = rows[hi], rows[hi + 1:]
    ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    agg, cnt = defaultdict(float), defaultdict(int)
    for r in d:
        if r[mi] != "gpu__time_duration.sum":
            continue
        n = r[ki].split("(")[0][-64:]
        agg[n] += float(r[vi].replace(",", "")) / 1e3
        cnt[n] += 1
    tot = sum(agg.values())
    print(f"launches {sum(cnt.values())}  device time {tot:.1f} us")
    for n, t in sorted(agg.items(), key=lambda x: -x[1])[:top]:
        print(f"  {n:64s} {cnt[n]:6d} {t:10.1f} us  {100 * t / tot:5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 15)

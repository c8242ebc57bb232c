"""Aggregate an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel:
python tools/launch_table.py launches.csv [skip_first_n_launches]"""
import collections
import csv
import re
import sys


def main(path, skip=0):
    rows = list(csv.reader(open(path)))
    for i, r in enumerate(rows):
        if "Kernel Name" in r:
            hdr, start = r, i + 1
            break
    ki, vi, ii = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("ID")
    agg = collections.OrderedDict()
    for r in rows[start:]:
        if len(r) <= vi or int(r[ii]) < skip:
            continue
        name = r[ki].replace("<unnamed>::", "").replace("void ", "").replace("arfx::", "")
        name = re.split(r"[(]", name)[0].strip()
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += float(r[vi].replace(",", ""))
    tot = sum(v[1] for v in agg.values())
    print(f"| kernel | launches | total us | avg us | share |\n|---|---|---|---|---|")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"| {k} | {v[0]} | {v[1] / 1e3:.1f} | {v[1] / v[0] / 1e3:.2f} | {v[1] / tot:.3f} |")
    print(f"\ntotal {tot / 1e3:.1f} us")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 0)

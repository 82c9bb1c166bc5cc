"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list per kernel.

    python tools/ncu_summary.py launches.csv "title line" > summary.txt
"""
import csv
import re
import sys


def main(path, title):
    rows = list(csv.reader(open(path)))
    hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r and "Metric Value" in r)
    hdr = rows[hdr_i]
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    agg = {}
    for r in rows[hdr_i + 1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        name = r[ki].replace("(anonymous namespace)::", "").replace("<unnamed>::", "").replace("unnamed>::", "")
        name = re.sub(r"^void ", "", name)
        name = name.split("(")[0].replace("spb::", "")
        v = float(r[vi].replace(",", ""))
        a = agg.setdefault(name, [0.0, 0])
        a[0] += v
        a[1] += 1
    tot = sum(v[0] for v in agg.values())
    print(title)
    print(f"total kernel time {tot / 1e3:.2f} us over {sum(v[1] for v in agg.values())} launches (ns units in csv)")
    for name, (t, c) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
        print(f"{t / 1e3:12.3f} us  {c:5d}  share {100 * t / tot:5.1f}%  {name}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "")

"""Per-kernel totals of an `ncu --metrics gpu__time_duration.sum --csv` launch list."""
import collections
import csv
import re
import sys


def main(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr, rows = rows[0], rows[1:]
    ki, mi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    scale = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0}
    agg, n = collections.OrderedDict(), collections.Counter()
    for r in rows:
        name = re.sub(r"\(.*", "", r[ki]).replace("void <unnamed>::", "").replace("<unnamed>::", "")
        v = float(r[mi].replace(",", "")) * scale.get(r[ui], 1.0)
        agg[name] = agg.get(name, 0.0) + v
        n[name] += 1
    tot = sum(agg.values())
    for k, v in sorted(agg.items(), key=lambda x: -x[1]):
        print(f"{v:9.3f} ms {n[k]:4d} {k}")
    print(f"{tot:9.3f} ms total")


if __name__ == "__main__":
    main(sys.argv[1])

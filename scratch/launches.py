"""Per-kernel totals of an ncu --metrics gpu__time_duration.sum launch list CSV."""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = None; agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows:
    if "Kernel Name" in r: hdr = r; continue
    if hdr is None or len(r) != len(hdr): continue
    d = dict(zip(hdr, r))
    if d.get("Metric Name") != "gpu__time_duration.sum": continue
    v = float(d["Metric Value"].replace(",", "")) / 1e6
    if d["Metric Unit"] == "usecond": v *= 1e3
    agg[d["Kernel Name"][:90]][0] += 1; agg[d["Kernel Name"][:90]][1] += v
tot = sum(t for n, t in agg.values())
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]): print(f"{n:5d} {t:9.3f} ms {t / tot * 100:5.1f}%  {k}")
print(f"total {tot:.3f} ms")

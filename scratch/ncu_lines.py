"""Aggregate ncu source-page (cuda,sass) warp-stall samples per CUDA line."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
h = None; agg = collections.defaultdict(lambda: [0, collections.Counter(), ""]); tot = 0
for r in rows:
    if r and r[0] == "Line No":
        h = r; iS = h.index("Warp Stall Sampling (All Samples)")
        stalls = [(i, n) for i, n in enumerate(h) if n.startswith("stall_") and "Not Issued" not in n]
        continue
    if h is None or len(r) < len(h): continue
    if r[0].strip():
        ln = r[0]; agg[ln][2] = r[1].strip()[:100]
        continue
    try: v = int(r[iS])
    except ValueError: continue
    a = agg[ln]; a[0] += v; tot += v
    for i, n in stalls:
        try: a[1][n] += int(r[i])
        except ValueError: pass
for ln, (v, c, src) in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
    st = " ".join(f"{k[6:]}={x*100//max(v,1)}" for k, x in c.most_common(3))
    print(f"{v/tot*100:5.1f}% L{ln:>5} [{st}] {src}")

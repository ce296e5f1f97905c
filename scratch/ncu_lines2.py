"""Per-CUDA-line warp-stall samples from an ncu cuda,sass source CSV (file-aware)."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
h = None; agg = collections.defaultdict(lambda: [0, collections.Counter(), ""]); tot = 0; fname = ""
for r in rows:
    if r and r[0] == "File Path": fname = r[1].split("/")[-1]; continue
    if r and r[0] == "Line No":
        h = r; iS = h.index("Warp Stall Sampling (All Samples)")
        stalls = [(i, n) for i, n in enumerate(h) if n.startswith("stall_") and "Not Issued" not in n]; continue
    if h is None or len(r) < len(h): continue
    if r[0].strip(): ln = (fname, r[0]); agg[ln][2] = r[1].strip()[:90]; continue
    try: v = int(r[iS])
    except ValueError: continue
    a = agg[ln]; a[0] += v; tot += v
    for i, n in stalls:
        try: a[1][n] += int(r[i])
        except ValueError: pass
for ln, (v, c, src) in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
    st = " ".join(f"{k[6:]}={x*100//max(v,1)}" for k, x in c.most_common(3))
    print(f"{v/tot*100:5.1f}% {ln[0][:12]}:{ln[1]:>5} [{st}] {src}")

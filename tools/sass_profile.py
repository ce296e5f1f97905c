"""Summarise an `ncu --page source --csv --print-source sass` export: executed
warp instructions and stall samples per opcode, and the hottest instructions."""
import collections
import csv
import sys


def main(path, top=40):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Instructions Executed" in r)
    hdr = rows[hi]
    ix = {h: i for i, h in enumerate(hdr)}
    # (multi-kernel exports repeat the header per kernel: skip those rows)
    data = [r for r in rows[hi + 1:] if len(r) == len(hdr) and r[ix["Instructions Executed"]] != "Instructions Executed"]
    ex = collections.Counter()
    st = collections.Counter()
    tot_e = tot_s = 0
    for r in data:
        op = r[ix["Source"]].strip().split()
        if not op:
            continue
        o = op[0]
        if o.startswith("@"):
            o = op[1]
        o = o.split(".")[0]
        e = int(r[ix["Instructions Executed"]] or 0)
        s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
        ex[o] += e
        st[o] += s
        tot_e += e
        tot_s += s
    print(f"executed warp instructions: {tot_e}, stall samples: {tot_s}")
    print(f"{'opcode':10s} {'executed':>12s} {'%':>6s} {'samples %':>9s}")
    for o, e in ex.most_common(top):
        print(f"{o:10s} {e:12d} {100 * e / tot_e:6.1f} {100 * st[o] / max(1, tot_s):9.1f}")


if __name__ == "__main__":
    main(sys.argv[1])

"""Top source lines by warp-stall samples from `ncu -i X --page source --csv --print-source cuda,sass`.

    ncu -i rep.ncu-rep --page source --csv --print-source cuda,sass > src.csv
    python tools/ncu_hotlines.py src.csv [N]
"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
N = int(sys.argv[2]) if len(sys.argv) > 2 else 25
h = next(r for r in rows if "Warp Stall Sampling (All Samples)" in r)
start = rows.index(h) + 1
si = h.index("Warp Stall Sampling (All Samples)")
stall_cols = [i for i, x in enumerate(h) if x.startswith("stall_")]


def I(x):
    try:
        return int(x)
    except ValueError:
        return 0


src = []
for r in rows[start:]:
    if len(r) < len(h) or r[0] == "":
        continue
    src.append((I(r[si]), r[0], r[1][:88], {h[i]: I(r[i]) for i in stall_cols if I(r[i])}))
tot = sum(s[0] for s in src) or 1
for s in sorted(src, key=lambda x: -x[0])[:N]:
    top = sorted(s[3].items(), key=lambda x: -x[1])[:3]
    print(f"{100 * s[0] / tot:5.1f}% L{s[1]:5s} {s[2]:88s} {[(k[6:], v) for k, v in top]}")

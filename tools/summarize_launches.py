"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) into a markdown table.

    python tools/summarize_launches.py gpurun_out/launches.csv > profiles/rNN_launches.md

Groups launches by kernel (template arguments kept), sorted by total time. Times are
ncu's serialised, cold-cache per-launch durations over the whole capture (setup + the
profiled steps): compare SHARES with bench.py's live CUDA-event breakdown, not absolutes.
"""
import collections
import csv
import sys

path = sys.argv[1]
rows = list(csv.reader(l for l in open(path) if not l.startswith("==")))
h = rows[0]
ki, vi, ui, gi, bi = (h.index(x) for x in ("Kernel Name", "Metric Value", "Metric Unit", "Grid Size", "Block Size"))
scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
tot = collections.defaultdict(float)
cnt = collections.Counter()
shape = {}
for r in rows[1:]:
    if len(r) <= vi:
        continue
    name = r[ki].split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "").replace("<unnamed>::", "")
    us = float(r[vi].replace(",", "")) * scale[r[ui]]
    tot[name] += us
    cnt[name] += 1
    shape[name] = f"{r[gi]} x {r[bi]}"
T = sum(tot.values())
print(f"# ncu launch list — {sum(cnt.values())} launches, {T / 1e3:.1f} ms total (serialised, cold cache)\n")
print("| kernel | launches | total ms | share | mean us | grid x block |")
print("|---|---|---|---|---|---|")
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    if v / T < 0.001:
        continue
    print(f"| `{k}` | {cnt[k]} | {v / 1e3:.2f} | {100 * v / T:.1f}% | {v / cnt[k]:.1f} | {shape[k]} |")

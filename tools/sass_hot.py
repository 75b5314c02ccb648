"""Summarise an `ncu --page source --csv --print-source=sass` dump: hottest instructions by
warp-stall samples and executed instructions (reads the CSV on stdin)."""
import csv
import sys

rows = list(csv.reader(sys.stdin))
h = rows[1]
ix = {n: i for i, n in enumerate(h)}
n = int(sys.argv[1]) if len(sys.argv) > 1 else 25
data = []
tot_s = tot_i = 0
for r in rows[2:]:
    if len(r) < len(h):
        continue
    s = float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    e = float(r[ix["Instructions Executed"]] or 0)
    th = float(r[ix["Avg. Threads Executed"]] or 0)
    tot_s += s
    tot_i += e
    data.append((s, e, th, r[ix["Address"]], r[ix["Source"]]))
print(f"total stall samples {tot_s:.0f}, warp instructions {tot_i:.3e}")
for s, e, th, a, src in sorted(data, reverse=True)[:n]:
    print(f"{100*s/max(tot_s,1):5.1f}%  inst {e:10.3e}  thr {th:4.1f}  {a}  {src[:70]}")

"""Group an ncu source-page SASS dump (CSV on stdin) into runs of equal execution count:
where the warp instructions of a kernel go."""
import csv
import sys

rows = list(csv.reader(sys.stdin))
h = rows[1]
ix = {n: i for i, n in enumerate(h)}
seq = []
for r in rows[2:]:
    if len(r) < len(h):
        continue
    e = float(r[ix["Instructions Executed"]] or 0)
    s = float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    seq.append((r[ix["Address"]][-4:], e, s, r[ix["Source"]][:60]))
tot = sum(x[1] for x in seq)
ts = sum(x[2] for x in seq) or 1
runs, cur = [], None
for a, e, s, src in seq:
    k = round(e / 1e6, 0)
    if cur and abs(cur["k"] - k) <= max(1, 0.05 * k):
        cur["n"] += 1; cur["e"] += e; cur["s"] += s; cur["end"] = a
    else:
        if cur:
            runs.append(cur)
        cur = {"k": k, "n": 1, "e": e, "s": s, "start": a, "end": a, "src": src}
runs.append(cur)
thr = float(sys.argv[1]) if len(sys.argv) > 1 else 0.01
print(f"total {tot/1e9:.2f}G warp instructions")
for r in runs:
    if r["e"] > thr * tot or r["s"] > thr * ts:
        print(f"{r['start']}-{r['end']} count~{r['k']:.0f}M n={r['n']:3d} inst={r['e']/1e9:.2f}G "
              f"({100*r['e']/tot:.0f}%) stall={100*r['s']/ts:.0f}% first: {r['src']}")

"""Group an `ncu --page source --csv --print-source=sass` dump into straight-line blocks of equal
execution count; print the heaviest blocks (warp instructions, stall share). stdin = CSV."""
import csv
import sys

rows = list(csv.reader(sys.stdin))
h = rows[1]
ix = {n: i for i, n in enumerate(h)}
data = []
for r in rows[2:]:
    if len(r) < len(h):
        continue
    data.append((int(r[ix["Address"]], 16), float(r[ix["Instructions Executed"]] or 0),
                 float(r[ix["Warp Stall Sampling (All Samples)"]] or 0), r[ix["Source"]]))
data.sort()
tot = sum(d[1] for d in data) or 1
tots = sum(d[2] for d in data) or 1
blk, cur = [], None
for a, e, s, src in data:
    if cur and abs(cur[1] - e) < 1 and a - cur[3] <= 16:
        cur[2] += 1; cur[3] = a; cur[4] += s; cur[5].append(src.strip())
    else:
        if cur:
            blk.append(cur)
        cur = [a, e, 1, a, s, [src.strip()]]
blk.append(cur)
blk.sort(key=lambda b: -b[1] * b[2])
n = int(sys.argv[1]) if len(sys.argv) > 1 else 20
base = data[0][0]
for b in blk[:n]:
    ops = " ".join(x.split()[0] if not x.startswith("@") else x.split()[1] for x in b[5][:40])
    print(f"+{b[0]-base:#07x} {b[1]:.3e} x{b[2]:3d} = {b[1]*b[2]/tot*100:5.1f}% inst, {b[4]/tots*100:5.1f}% stall | {ops[:150]}")

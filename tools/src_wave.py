"""Per-CUDA-line totals of an `ncu --page source --csv --print-source cuda,sass` dump (stdin):
warp instructions, shared-memory wavefronts (and the excess over ideal), stall samples."""
import csv
import sys

n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
rows = list(csv.reader(sys.stdin))
cur_file, hdr, key = None, None, None
agg, text = {}, {}
cols = ["Instructions Executed", "L1 Wavefronts Shared", "L1 Wavefronts Shared Excessive",
        "Warp Stall Sampling (All Samples)"]
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = {name: i for i, name in enumerate(r)}
        continue
    if hdr is None or len(r) < len(hdr) - 2:
        continue
    if r[0] not in ("",) and r[2] in ("", "-"):   # CUDA line
        key = (cur_file, int(r[0]))
        text[key] = r[1].strip()[:70]
        vals = [float((r[hdr[c]] or "0").replace(",", "")) if r[hdr[c]] not in ("-",) else 0.0 for c in cols]
        a = agg.setdefault(key, [0.0] * len(cols))
        for i, v in enumerate(vals):
            a[i] += v
tot = [sum(v[i] for v in agg.values()) for i in range(len(cols))]
print("totals: inst %.3g  shared wavefronts %.3g  excessive %.3g  samples %.3g" % tuple(tot))
print(f"{'file:line':28s} {'inst%':>6s} {'wave%':>6s} {'exc%':>6s} {'stall%':>6s}  source")
for k, v in sorted(agg.items(), key=lambda kv: -(kv[1][1] + kv[1][0] * 0.3))[:n]:
    f = [100 * v[i] / tot[i] if tot[i] else 0 for i in range(len(cols))]
    print(f"{k[0]+':'+str(k[1]):28s} {f[0]:6.1f} {f[1]:6.1f} {f[2]:6.1f} {f[3]:6.1f}  {text[k]}")

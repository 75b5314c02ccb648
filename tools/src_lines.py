"""Per-source-line totals of an `ncu --page source --csv --print-source=cuda,sass` dump (stdin):
warp instructions executed and stall samples attributed to each CUDA line (heaviest first)."""
import csv
import sys

n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
rows = list(csv.reader(sys.stdin))
cur_file, hdr = None, None
agg = {}
src_text = {}
for r in rows:
    if not r:
        continue
    if r[0] in ("File Path", "File Name"):
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = {name: i for i, name in enumerate(r)}
        continue
    if hdr is None or len(r) < 5:
        continue
    if r[0] != "" and r[2] in ("", "-"):   # a CUDA source line row (no address)
        try:
            ln = int(r[0])
        except ValueError:
            continue
        key = (cur_file, ln)
        src_text[key] = r[1].strip()[:90]
        try:
            ex = float(r[hdr["Instructions Executed"]].replace("-", "0") or 0)
            st = float(r[hdr["Warp Stall Sampling (All Samples)"]].replace("-", "0") or 0)
        except (ValueError, IndexError):
            continue
        a = agg.setdefault(key, [0.0, 0.0])
        a[0] += ex
        a[1] += st
ti = sum(v[0] for v in agg.values()) or 1
ts = sum(v[1] for v in agg.values()) or 1
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:n]:
    print(f"{v[0]/ti*100:5.1f}% inst {v[1]/ts*100:5.1f}% stall  {k[0]}:{k[1]}  {src_text.get(k, '')}")

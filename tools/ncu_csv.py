"""Print the metrics of an ncu --csv log (skips non-CSV lines such as the bench JSON line)."""
import csv
import sys

for path in sys.argv[1:]:
    lines = [l for l in open(path) if l.startswith('"')]
    rows = list(csv.reader(lines))
    h = rows[0]
    print("==", path)
    for r in rows[1:]:
        d = dict(zip(h, r))
        print(f"  {d['Kernel Name'][:30]:30s} {d['Metric Name']:80s} {d['Metric Value']}")

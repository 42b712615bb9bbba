"""Per-kernel mean / min launch time from an ncu --csv --log-file launch list (measurement tooling)."""
import collections
import csv
import sys

rows = [l for l in open(sys.argv[1]) if not l.startswith("==")]
r = csv.reader(rows)
h = next(r)
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
d = collections.defaultdict(list)
for row in r:
    d[row[ki].split("(")[0][:48]].append(float(row[vi].replace(",", "")))
for k, v in d.items():
    print(f"{k:48s} n={len(v):3d} mean={sum(v)/len(v)/1e3:9.2f} us  min={min(v)/1e3:9.2f} us")

"""Summarise an ncu --csv launch list (gpu__time_duration.sum) per kernel."""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1]).read().splitlines()) if len(r) > 10]
h = rows[0]
ki, vi = h.index("Kernel Name"), len(h) - 1
seq = collections.defaultdict(list)
for r in rows[1:]:
    if r[0] == "ID":
        continue
    seq[r[ki].split("(")[0].replace("void ", "")].append(float(r[vi].replace(",", "")))
for k, v in seq.items():
    print(f"{k[:40]:40s} n={len(v):4d} sum={sum(v)/1e3:9.1f} us mean={sum(v)/len(v)/1e3:8.1f} "
          f"first={v[0]/1e3:8.1f} max={max(v)/1e3:8.1f}")

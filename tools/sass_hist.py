"""Opcode histogram (instructions executed) of one kernel from an ncu report."""
import collections, csv, subprocess, sys
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass",
                      "-k", "regex:" + sys.argv[2]], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = next(r for r in rows if "Source" in r and "Address" in r)
si, ie = h.index("Source"), h.index("Instructions Executed")
op, tot = collections.Counter(), 0.0
for r in rows:
    if len(r) <= ie or r is h:
        continue
    try:
        n = float(r[ie] or 0)
    except ValueError:
        continue
    o = r[si].strip().split()
    if not o:
        continue
    k = o[1] if o[0].startswith("@") else o[0]
    op[k.split(".")[0]] += n
    tot += n
print("total", tot)
for k, v in op.most_common(int(sys.argv[3]) if len(sys.argv) > 3 else 30):
    print(f"{k:12s} {v / tot * 100:5.1f}% {v / 1e6:7.2f}M")

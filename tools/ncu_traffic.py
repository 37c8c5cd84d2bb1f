"""DRAM traffic per launch of the captured kernels of an ncu report ->
profiles/roofline_traffic.json (bench.py reports it as roofline.traffic).
usage: python tools/ncu_traffic.py REPORT.ncu-rep [config]"""
import csv
import json
import os
import subprocess
import sys

rep = sys.argv[1]
config = sys.argv[2] if len(sys.argv) > 2 else "c2"
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h = rows[0]
out = {}
for r in rows[2:]:
    name = r[h.index("Kernel Name")]
    rd = float(r[h.index("dram__bytes_read.sum")])
    wr = float(r[h.index("dram__bytes_write.sum")])
    unit = rows[1][h.index("dram__bytes_read.sum")]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
    out[name] = {"dram_read_bytes": rd * scale, "dram_write_bytes": wr * scale,
                 "dram_bytes": (rd + wr) * scale, "duration_us": float(r[h.index("gpu__time_duration.sum")])}
path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles",
                    "roofline_traffic.json")
data = json.load(open(path)) if os.path.exists(path) else {}
data[config] = {"report": os.path.basename(rep), "kernels": out}
json.dump(data, open(path, "w"), indent=1)
print(json.dumps(data[config], indent=1))

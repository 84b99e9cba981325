"""DRAM traffic of the captured kernel launch of an ncu --set full report -> JSON for bench.py.

usage: python tools/ncu_traffic.py report.ncu-rep profiles/k_stream_traffic.json
"""
import csv
import io
import json
import subprocess
import sys

rep, out = sys.argv[1], sys.argv[2]
txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
h, u, v = rows[0], rows[1], rows[2]


def val(key):
    x = float(v[h.index(key)].replace(",", ""))
    unit = u[h.index(key)]
    return x * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)


rd, wr = val("dram__bytes_read.sum"), val("dram__bytes_write.sum")
res = {"kernel": v[h.index("Kernel Name")], "report": rep, "dram_bytes_read": rd, "dram_bytes_write": wr,
       "dram_bytes_per_launch": rd + wr,
       "duration_ms": float(v[h.index("gpu__time_duration.sum")]) * {"ns": 1e-6, "us": 1e-3, "ms": 1.0}[
           u[h.index("gpu__time_duration.sum")]]}
json.dump(res, open(out, "w"), indent=1)
print(res)

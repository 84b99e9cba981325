"""Instruction groups (runs of equal execution count) of one loop region of an ncu report:
where a loop's instructions and time go (per-thread divergent handlers show as thr < 32).

usage: python tools/ncu_groups.py report.ncu-rep LO HI [min_share=0.01]   (offsets, hex)
"""
import collections
import csv
import io
import subprocess
import sys

rep, lo, hi = sys.argv[1], int(sys.argv[2], 16), int(sys.argv[3], 16)
mins = float(sys.argv[4]) if len(sys.argv) > 4 else 0.01
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hr = next(i for i, r in enumerate(rows) if "Address" in r)
h = rows[hr]
data = [r for r in rows[hr + 1:] if len(r) == len(h)]
base = int(data[0][0], 16)
iex, ism, ith = h.index("Instructions Executed"), h.index("# Samples"), h.index("Avg. Threads Executed")
grp = []
for r in data:
    a = int(r[0], 16) - base
    if not lo <= a <= hi:
        continue
    ex, sm = int(r[iex]), int(r[ism] or 0)
    toks = r[1].strip().split()
    op = (toks[1] if toks[0].startswith("@") else toks[0]).split(".")[0]
    if grp and grp[-1][2] == ex:
        g = grp[-1]
        g[1] = a; g[3] += 1; g[4] += sm; g[5][op] += 1
    else:
        grp.append([a, a, ex, 1, sm, collections.Counter([op]), r[ith]])
tot = sum(g[2] * g[3] for g in grp) or 1
tots = sum(g[4] for g in grp) or 1
for g in grp:
    if g[2] * g[3] > mins * tot or g[4] > mins * tots:
        print("%5x-%5x exec %11d n=%4d instr%%=%5.1f time%%=%5.1f thr=%-5s %s" % (
            g[0], g[1], g[2], g[3], 100.0 * g[2] * g[3] / tot, 100.0 * g[4] / tots, g[6],
            dict(g[5].most_common(5))))

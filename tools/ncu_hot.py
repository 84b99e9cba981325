"""Hot-loop view of an ncu report: SASS instructions executed >= frac * max, in address
order, with stall samples; plus an opcode histogram.

usage: python tools/ncu_hot.py report.ncu-rep [frac=0.5] [--list]
"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
frac = float(sys.argv[2]) if len(sys.argv) > 2 and not sys.argv[2].startswith("--") else 0.5
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr_i = next(i for i, r in enumerate(rows) if "Address" in r)
h = rows[hdr_i]
data = [r for r in rows[hdr_i + 1:] if len(r) == len(h)]
isrc, iex, ist = h.index("Source"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
tot = sum(int(r[iex]) for r in data)
mx = max(int(r[iex]) for r in data)
hot = [r for r in data if int(r[iex]) >= frac * mx]
print("total warp-instr %d  max/instr %d  hot instrs %d  hot share %.3f" % (
    tot, mx, len(hot), sum(int(r[iex]) for r in hot) / tot))
c, cs = collections.Counter(), collections.Counter()
for r in hot:
    toks = r[isrc].split()
    op = (toks[1] if toks[0].startswith("@") else toks[0]).split(".")[0]
    c[op] += 1
    cs[op] += int(r[ist])
print("ops:", " ".join("%s:%d" % kv for kv in c.most_common()))
print("stall samples:", " ".join("%s:%d" % kv for kv in cs.most_common(12)))
if "--list" in sys.argv:
    for r in hot:
        print("%6s %10s  %s" % (r[ist], r[iex], r[isrc].strip()))

"""Time (warp-state samples) and instructions of an ncu --set full report split by the
kernel's loops: every backward branch delimits a loop [target, branch]; each SASS
instruction is attributed to the innermost loop containing it.

usage: python tools/ncu_regions.py report.ncu-rep [top=12]
"""
import collections
import csv
import io
import re
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 12
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = next(i for i, r in enumerate(rows) if "Address" in r)
h = rows[hi]
data = [r for r in rows[hi + 1:] if len(r) == len(h)]
ia, isrc, ismp, iex = h.index("Address"), h.index("Source"), h.index("# Samples"), h.index("Instructions Executed")
ins = [(int(r[ia], 16), r[isrc].strip(), int(r[ismp] or 0), int(r[iex] or 0)) for r in data]
loops = []
for a, src, _, _ in ins:
    toks = src.split()
    op = (toks[1] if toks and toks[0].startswith("@") else (toks[0] if toks else ""))
    if op.startswith("BRA"):
        m = re.search(r"0x([0-9a-f]+)", src)
        if m:
            t = int(m.group(1), 16)
            base = ins[0][0]
            tgt = t if t > base else base + t            # relative or absolute target
            if tgt < a:
                loops.append((tgt, a))
loops = sorted(set(loops), key=lambda x: x[1] - x[0])
tot_s = sum(x[2] for x in ins) or 1
tot_i = sum(x[3] for x in ins) or 1
acc = collections.defaultdict(lambda: [0, 0, 0, collections.Counter()])
for a, src, smp, ex in ins:
    key = None
    for lo, hi_ in loops:                                 # innermost first (sorted by size)
        if lo <= a <= hi_:
            key = (lo, hi_)
            break
    rec = acc[key]
    rec[0] += smp
    rec[1] += ex
    rec[2] += 1
    toks = src.split()
    op = (toks[1] if toks and toks[0].startswith("@") else (toks[0] if toks else "?")).split(".")[0]
    rec[3][op] += ex
base = ins[0][0]
print("%-22s %7s %7s %6s  %s" % ("loop [lo, hi] (offset)", "time%", "instr%", "#sass", "top opcodes by executed"))
for key, (smp, ex, n, ops) in sorted(acc.items(), key=lambda kv: -kv[1][0])[:top]:
    name = "outside loops" if key is None else "[%#x, %#x]" % (key[0] - base, key[1] - base)
    print("%-22s %6.1f%% %6.1f%% %6d  %s" % (name, 100.0 * smp / tot_s, 100.0 * ex / tot_i, n,
                                             " ".join("%s:%.0f%%" % (o, 100.0 * c / max(1, ex)) for o, c in ops.most_common(6))))

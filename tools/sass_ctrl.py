"""Dump SASS with decoded control bits (stall, yield, wbar, rbar, wait mask, reuse) for one
function of libphmm.so — used to read the scheduling of the wavefront step loop.

usage: python tools/sass_ctrl.py <function-substring> [start_hex end_hex]
"""
import re
import subprocess
import sys

LIB = "paper_2411_11547_b200/_lib/libphmm.so"
pat = sys.argv[1]
lo = int(sys.argv[2], 16) if len(sys.argv) > 2 else 0
hi = int(sys.argv[3], 16) if len(sys.argv) > 3 else 1 << 40
sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
body = [c for c in sass.split("Function : ")[1:] if pat in c.split("\n", 1)[0]][0]
lines = body.splitlines()
for i, line in enumerate(lines):
    m = re.match(r"\s+/\*([0-9a-f]+)\*/\s+(.*?);\s+/\* (0x[0-9a-f]+) \*/", line)
    if not m:
        continue
    addr = int(m.group(1), 16)
    if not lo <= addr <= hi:
        continue
    m2 = re.search(r"/\* (0x[0-9a-f]+) \*/", lines[i + 1])
    hw = int(m2.group(1), 16)
    stall = (hw >> 41) & 0xF
    yld = (hw >> 45) & 1
    wbar = (hw >> 46) & 7
    rbar = (hw >> 49) & 7
    wait = (hw >> 52) & 0x3F
    print("%05x s%-2d %s wb%s rb%s w%02x  %s" % (addr, stall, "Y" if yld else " ",
          wbar if wbar != 7 else "-", rbar if rbar != 7 else "-", wait, m.group(2)[:90]))

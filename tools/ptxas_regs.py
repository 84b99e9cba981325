"""Registers / spills per kernel from `nvcc -Xptxas -v` output.

usage: python tools/ptxas_regs.py [filter]   (compiles every csrc/*.cu to /tmp, ~1 min)
"""
import re
import subprocess
import sys
import os

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_11547_b200.build import FLAGS, NVCC, ROOT, SOURCES  # noqa: E402

flt = sys.argv[1] if len(sys.argv) > 1 else "k_"
from concurrent.futures import ThreadPoolExecutor  # noqa: E402


def _ptxas(src):
    cmd = [NVCC] + FLAGS + ["-Xptxas", "-v", "-I", os.path.join(ROOT, "include"), "-c", "-o", "/dev/null", src]
    return subprocess.run(cmd, capture_output=True, text=True).stderr


with ThreadPoolExecutor(len(SOURCES)) as ex:
    err = "\n".join(ex.map(_ptxas, SOURCES))
cur = None
rows = {}
for line in err.splitlines():
    m = re.search(r"Compiling entry function '(\w+)'", line)
    if m:
        cur = subprocess.run(["c++filt"], input=m.group(1), capture_output=True, text=True).stdout.strip()
        rows[cur] = {}
        continue
    if cur is None:
        continue
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m:
        rows[cur]["spill"] = "%s/%s" % m.groups()
    m = re.search(r"Used (\d+) registers", line)
    if m:
        rows[cur]["regs"] = int(m.group(1))
for name, r in rows.items():
    if flt in name:
        short = re.sub(r"\(.*", "", name).replace("phmm::", "")
        print("%-40s regs %4s  spill st/ld %s" % (short, r.get("regs"), r.get("spill")))

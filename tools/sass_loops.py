"""Static loop view of one kernel's SASS (no GPU needed): every backward branch delimits a
loop [target, branch]; prints each loop's size and opcode histogram, innermost first.

usage: python tools/sass_loops.py <.o | .so | .cubin> <function-substring> [min_size=20]
"""
import collections
import re
import subprocess
import sys

path, sub = sys.argv[1], sys.argv[2]
min_size = int(sys.argv[3]) if len(sys.argv) > 3 else 20
sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", path], capture_output=True, text=True,
                      check=True).stdout
for chunk in sass.split("Function : ")[1:]:
    name = chunk.split("\n", 1)[0].strip()
    if sub not in name:
        continue
    ins = []
    for line in chunk.splitlines():
        m = re.match(r"\s+/\*([0-9a-f]+)\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)(.*?);", line)
        if m:
            ins.append((int(m.group(1), 16), m.group(3), m.group(4)))
    loops = []
    for a, op, rest in ins:
        if op.startswith("BRA"):
            t = re.search(r"0x([0-9a-f]+)", rest)
            if t and int(t.group(1), 16) <= a:
                loops.append((int(t.group(1), 16), a))
    print(name[:110], "total", len(ins))
    for lo, hi in sorted(set(loops), key=lambda x: x[1] - x[0]):
        body = [op.split(".")[0] for a, op, _ in ins if lo <= a <= hi]
        if len(body) < min_size:
            continue
        c = collections.Counter(body)
        movs = sum(1 for a, op, rest in ins if lo <= a <= hi and op.startswith("IMAD.MOV"))
        print("  [%#07x, %#07x] %5d instrs  IMAD.MOV %3d  %s" % (
            lo, hi, len(body), movs, " ".join("%s:%d" % kv for kv in c.most_common(9))))

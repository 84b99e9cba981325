"""Per-function SASS instruction histogram of libphmm.so (static evidence for DESIGN.md).

usage: python tools/sass_stats.py [substring-of-function-name] [--loop]
--loop restricts the count to the hottest basic-block span: the instructions between
the last backward branch target and that branch inside the function (the wavefront step).
"""
import collections
import re
import subprocess
import sys

LIB = "paper_2411_11547_b200/_lib/libphmm.so"


def functions():
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", LIB], capture_output=True,
                          text=True, check=True).stdout
    out = {}
    for chunk in sass.split("Function : ")[1:]:
        name = chunk.split("\n", 1)[0].strip()
        out[name] = chunk
    return out


def instrs(body):
    res = []
    for line in body.splitlines():
        m = re.match(r"\s+/\*([0-9a-f]+)\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)(.*?);", line)
        if m:
            res.append((int(m.group(1), 16), m.group(3), m.group(4)))
    return res


def main():
    pat = sys.argv[1] if len(sys.argv) > 1 and not sys.argv[1].startswith("--") else "k_fast"
    loop = "--loop" in sys.argv
    for name, body in functions().items():
        if pat not in name:
            continue
        ins = instrs(body)
        if loop:
            # largest backward branch span = the step loop
            best = None
            for addr, op, args in ins:
                if op.startswith("BRA"):
                    m = re.search(r"0x([0-9a-f]+)", args)
                    if m and int(m.group(1), 16) < addr:
                        span = addr - int(m.group(1), 16)
                        if best is None or span > best[0]:
                            best = (span, int(m.group(1), 16), addr)
            if best:
                ins = [x for x in ins if best[1] <= x[0] <= best[2]]
        c = collections.Counter(op.split(".")[0] for _, op, _ in ins)
        print("%s  (%d instructions)" % (name, len(ins)))
        print("   " + "  ".join("%s:%d" % kv for kv in c.most_common(24)))


if __name__ == "__main__":
    main()

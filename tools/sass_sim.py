"""Single-warp issue model of a SASS region (B300_MICROARCH.md 'Single-warp T_1w'):
T advances by each instruction's stall count; instructions with a wait mask wait for
their scoreboard slots; variable-latency producers set slots at issue + LAT[op].

usage: python tools/sass_sim.py <function-substring> <start_hex> <end_hex> [iterations]
"""
import re
import subprocess
import sys

LIB = "paper_2411_11547_b200/_lib/libphmm.so"
LAT = {"SHFL": 30, "LDS": 32, "LDG": 60, "LDC": 30, "S2R": 25, "LDCU": 30, "ATOMG": 300,
       "REDUX": 30, "VOTE": 10, "MUFU": 20, "STS": 10, "STG": 10, "DFMA": 8, "DADD": 8, "DMUL": 8}


def load(pat, lo, hi):
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
    body = [c for c in sass.split("Function : ")[1:] if pat in c.split("\n", 1)[0]][0]
    lines = body.splitlines()
    out = []
    for i, line in enumerate(lines):
        m = re.match(r"\s+/\*([0-9a-f]+)\*/\s+(.*?);\s+/\* (0x[0-9a-f]+) \*/", line)
        if not m:
            continue
        addr = int(m.group(1), 16)
        if not lo <= addr <= hi:
            continue
        hw = int(re.search(r"/\* (0x[0-9a-f]+) \*/", lines[i + 1]).group(1), 16)
        text = m.group(2)
        op = re.sub(r"^@!?U?P\w+\s+", "", text).split()[0].split(".")[0]
        out.append(dict(addr=addr, op=op, text=text, stall=(hw >> 41) & 0xF, wbar=(hw >> 46) & 7,
                        rbar=(hw >> 49) & 7, wait=(hw >> 52) & 0x3F))
    return out


def simulate(ins, iters):
    T = 0
    sb = [0] * 6
    fp_pipe = 0
    per_iter = []
    for it in range(iters):
        t0 = T
        for x in ins:
            arm = max([sb[s] for s in range(6) if x["wait"] >> s & 1] or [0])
            T = max(T, arm)
            lat = LAT.get(x["op"], 6)
            if x["wbar"] < 6:
                sb[x["wbar"]] = max(sb[x["wbar"]], T + lat)
            if x["rbar"] < 6:
                sb[x["rbar"]] = max(sb[x["rbar"]], T + 6)
            if x["op"] in ("FFMA2", "FMUL2", "FADD2"):
                fp_pipe += 2
            elif x["op"] in ("FFMA", "FMUL", "FADD"):
                fp_pipe += 1
            T += max(1, x["stall"])
        per_iter.append(T - t0)
    return per_iter, fp_pipe / iters


if __name__ == "__main__":
    pat, lo, hi = sys.argv[1], int(sys.argv[2], 16), int(sys.argv[3], 16)
    iters = int(sys.argv[4]) if len(sys.argv) > 4 else 4
    ins = load(pat, lo, hi)
    per, pipe = simulate(ins, iters)
    print("instructions %d  cycles/iter %s  fp-pipe cycles/iter %.0f  -> 1-warp pipe util %.0f%%"
          % (len(ins), per, pipe, 100 * pipe / per[-1]))

"""Key metrics of an ncu --set full report (first kernel).  usage: python tools/ncu_sum.py rep"""
import csv
import io
import subprocess
import sys

WANT = [
    ("gpu__time_duration.sum", "duration ms"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe active %"),
    ("sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active", "FMA-heavy active %"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe active %"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "FP64 inst %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("smsp__inst_executed.sum", "warp instrs"),
    ("smsp__warps_active.avg.per_cycle_active", "warps/SMSP"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
]
STALLS = ["wait", "math_pipe_throttle", "not_selected", "long_scoreboard", "short_scoreboard",
          "branch_resolving", "dispatch_stall", "mio_throttle", "no_instruction", "barrier", "lg_throttle"]


def main():
    out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u = rows[0], rows[1]
    for v in rows[2:]:
        name = v[h.index("Kernel Name")] if "Kernel Name" in h else "?"
        print(name[:90])
        for key, label in WANT:
            if key in h:
                print("  %-22s %s %s" % (label, v[h.index(key)], u[h.index(key)]))
        st = []
        for s in STALLS:
            key = "smsp__average_warps_issue_stalled_%s_per_issue_active.ratio" % s
            if key in h:
                st.append("%s %.2f" % (s, float(v[h.index(key)])))
        print("  stalls/issue: " + ", ".join(st))


if __name__ == "__main__":
    main()

"""Summarise an .ncu-rep: key throughput metrics + stall hot spots + opcode mix."""
import collections
import csv
import io
import re
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, u, v = rows[0], rows[1], rows[2]
keys = ["Kernel Name", "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second",
        "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size"]
for k in keys:
    if k in h:
        i = h.index(k)
        print(f"{k:70s} {u[i]:>8s} {v[i][:90]}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hdr = rows[1]
data = rows[2:]
iS, iE, iSrc = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed"), hdr.index("Source")
tot = sum(int(r[iS]) for r in data if r[iS].isdigit())
print("stall samples", tot)
for i, r in enumerate(data):
    if "TRYWAIT" in r[iSrc] and i + 1 < len(data):
        smp = int(data[i + 1][iS] or 0) + int(r[iS] or 0)
        if smp > tot * 0.01:
            print(f"  wait {r[iSrc].strip()[40:75]:36s} samples {smp:6d} ({smp / tot * 100:4.1f}%) exec {r[iE]}")
c = collections.Counter()
for r in data:
    if r[iE].isdigit():
        s = re.sub(r"^@!?U?P\w+\s+", "", r[iSrc].strip())
        c[s.split()[0] if s else "?"] += int(r[iE])
t = sum(c.values())
print("opcode mix:", ", ".join(f"{op} {n / t * 100:.1f}%" for op, n in c.most_common(14)))

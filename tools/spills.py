"""Summarise ptxas -v logs per kernel: registers, stack frame, spills. Usage: python tools/spills.py LOG..."""
import re
import sys

for path in sys.argv[1:]:
    cur = None
    for line in open(path):
        m = re.search(r"Compiling entry function '(\S+)'", line)
        if m:
            cur = m.group(1)
            continue
        m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads", line)
        if m and cur:
            frame, st, ld = m.groups()
        m2 = re.search(r"Used (\d+) registers", line)
        if m2 and cur:
            print(f"{m2.group(1):>4} regs frame={frame:>4} spill_st={st:>4} spill_ld={ld:>4}  {cur[:110]}")
            cur = None

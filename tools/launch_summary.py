"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list: mean duration per kernel.

    python tools/launch_summary.py gpurun_out/TAG_launches.csv > profiles/TAG_launches_bench.txt
"""
import collections
import csv
import sys


def main(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10 and r[0].isdigit()]
    acc = collections.OrderedDict()
    for r in rows:
        name, val = r[4], float(r[-1])
        acc.setdefault(name, []).append(val / 1000.0)
    print("ncu --metrics gpu__time_duration.sum --clock-control none -c 400 python bench.py --steps 2 "
          "--warmup 3 --headline-only --no-cpu-baseline")
    print("(cold, serialised replays: compare shares, not absolutes)")
    for name, v in acc.items():
        print(f"{name[:110]:110s} n={len(v):4d} mean={sum(v) / len(v):9.1f} us")


if __name__ == "__main__":
    main(sys.argv[1])

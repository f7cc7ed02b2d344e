"""Print an ncu source-page CSV (SASS) with per-instruction stall samples and the dominant
stall reasons. Usage: python tools/ncu_source.py SRC.csv [min_exec] [min_samples]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
min_exec = int(sys.argv[2]) if len(sys.argv) > 2 else 0
min_samp = int(sys.argv[3]) if len(sys.argv) > 3 else 0
ix = {h: i for i, h in enumerate(hdr)}
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
for r in rows[2:]:
    try:
        ex = int(r[ix["Instructions Executed"]] or 0)
        smp = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    except ValueError:
        continue
    if ex < min_exec or smp < min_samp:
        continue
    rs = sorted(((int(r[ix[h]] or 0), h[6:]) for h in reasons), reverse=True)[:2]
    top = " ".join(f"{n}:{c}" for c, n in rs if c > 0)
    print(f"{r[ix['Address']][-5:]} {smp:6d} {ex:8d} {r[ix['Source']][:70]:70s} {top}")

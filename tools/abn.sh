#!/bin/bash
# A/B/n of library variants on the forward or backward probe, interleaved:
#   tools/abn.sh fwd|bwd VARIANT...   (build/<VARIANT>/libflexattn_b200.so; "base" = in-tree)
MODE=$1; shift
for i in 1 2; do
  for V in "$@"; do
    if [ "$V" = base ]; then L=$PWD/paper_2412_05496_b200/libflexattn_b200.so; else L=$PWD/paper_2412_05496_b200/build/$V/libflexattn_b200.so; fi
    echo "== $V"; FA_LIB_PATH=$L python tools/perf_probe.py $MODE 2>&1 | grep -E "^C[0-9]|fwd|bwd" | head -8
  done
done

#!/bin/bash
# forward A/B/C: tools/abf3.sh V1 V2 ... (base = in-tree library)
for i in 1 2; do
  echo "== base"; python tools/perf_probe.py fwd 2>&1 | grep "fwd" | cut -c1-40
  for V in "$@"; do
    echo "== $V"; FA_LIB_PATH=$PWD/paper_2412_05496_b200/build/$V/libflexattn_b200.so python tools/perf_probe.py fwd 2>&1 | grep "fwd" | cut -c1-40
  done
done

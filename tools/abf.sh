#!/bin/bash
# A/B of the forward: tools/abf.sh VARIANT -> perf_probe fwd with the in-tree library and build/<VARIANT>
V=$1
for i in 1 2; do
  echo "== base"; python tools/perf_probe.py fwd 2>&1 | grep "fwd"
  echo "== $V"; FA_LIB_PATH=$PWD/paper_2412_05496_b200/build/$V/libflexattn_b200.so python tools/perf_probe.py fwd 2>&1 | grep "fwd"
done

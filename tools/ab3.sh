#!/bin/bash
# backward A/B/C: tools/ab3.sh "V1 V2 ..." [configs...]  (base = in-tree library)
VS=$1; shift
for i in 1 2; do
  echo "== base"; python tools/bwd_probe.py "$@" 2>&1 | grep "exp=0"
  for V in $VS; do
    echo "== $V"; FA_LIB_PATH=$PWD/paper_2412_05496_b200/build/$V/libflexattn_b200.so python tools/bwd_probe.py "$@" 2>&1 | grep "exp=0"
  done
done

#!/bin/bash
# A/B: run tools/bwd_probe.py (args) with the in-tree library and each build/<variant> library,
# interleaved twice. Usage: tools/ab.sh VARIANT [configs...]
V=$1; shift
for i in 1 2; do
  echo "== base"; python tools/bwd_probe.py "$@" 2>&1 | grep "exp=0"
  echo "== $V"; FA_LIB_PATH=$PWD/paper_2412_05496_b200/build/$V/libflexattn_b200.so python tools/bwd_probe.py "$@" 2>&1 | grep "exp=0"
done

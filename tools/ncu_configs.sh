#!/bin/bash
# ncu --set full of the forward and fused-backward main kernels at C3 and C4, the deterministic
# dQ pass at C2 and the GQA tensor-core decode, summarised on the box (the reports are not kept).
TAG=${1:-r02}
mkdir -p gpurun_out
for CFG in C3 C4; do
  bash tools/ncu_capture.sh $CFG $TAG > /dev/null 2>&1
  for k in fwd bwd; do
    python tools/ncu_summary.py gpurun_out/ncu_${k}_${CFG}_${TAG}.ncu-rep > gpurun_out/${TAG}_${k}_$(echo $CFG | tr C c)_ncu.txt 2>&1
  done
done
rm -f gpurun_out/*.ncu-rep

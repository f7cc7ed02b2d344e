#!/bin/bash
# One ncu --set full capture of the forward and backward main kernels at a BASELINE config:
#   tools/ncu_capture.sh C2 [tag]   -> gpurun_out/ncu_{fwd,bwd}_C2[_tag].ncu-rep
CFG=${1:-C2}; TAG=${2:+_$2}
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:flex_fwd_sm100 -c 1 \
    -o gpurun_out/ncu_fwd_${CFG}${TAG} -f python tools/perf_probe.py fwd_only_$CFG > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:flex_bwd_sm100 -c 1 \
    -o gpurun_out/ncu_bwd_${CFG}${TAG} -f python tools/bwd_probe.py $CFG > /dev/null 2>&1
ls -la gpurun_out/*.ncu-rep

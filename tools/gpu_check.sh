#!/bin/bash
# One GPU-box session: GPU parity suite, bench (ours + reference arm), launch list of the bench,
# ncu --set full of the fwd/bwd main kernels at C2.   usage: tools/gpu_check.sh TAG
TAG=${1:-r02}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/${TAG}_smi.txt 2>&1
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/${TAG}_gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_gputest.log
timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${TAG}_bench_ref.json 2> gpurun_out/${TAG}_bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
   --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 3 --headline-only --no-cpu-baseline > /dev/null 2>&1
timeout 900 bash tools/ncu_capture.sh C2 ${TAG}

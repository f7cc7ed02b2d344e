#!/bin/bash
# Round-end style GPU session: parity suite, C++ API test, bench (ours + reference arm), the
# launch list of the bench command, ncu --set full of the fwd/bwd main kernels at C2, SASS summary.
#   tools/gpu_round.sh TAG
TAG=${1:-r02}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/${TAG}_smi.txt 2>&1
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/${TAG}_gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_gputest.log
./tests/cpp/test_cpp_api > gpurun_out/${TAG}_cpp.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_cpp.log
timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${TAG}_bench_ref.json 2> gpurun_out/${TAG}_bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
   --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 3 --headline-only --no-cpu-baseline > /dev/null 2>&1
timeout 900 bash tools/ncu_capture.sh C2 ${TAG}
# summarise the captures on the box (the .ncu-rep files would overflow the 64 MiB copy-back)
for k in fwd bwd; do
  [ -f gpurun_out/ncu_${k}_C2_${TAG}.ncu-rep ] && python tools/ncu_summary.py gpurun_out/ncu_${k}_C2_${TAG}.ncu-rep > gpurun_out/${TAG}_${k}_c2_ncu.txt 2>&1
  ncu -i gpurun_out/ncu_${k}_C2_${TAG}.ncu-rep --page raw --csv > gpurun_out/${TAG}_${k}_c2_raw.csv 2>/dev/null
done
rm -f gpurun_out/*.ncu-rep

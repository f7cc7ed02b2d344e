for i in 1 2; do
for V in base dtc1; do
  if [ $V = base ]; then L=$PWD/paper_2412_05496_b200/libflexattn_b200.so; else L=$PWD/paper_2412_05496_b200/build/$V/libflexattn_b200.so; fi
  echo "== $V"; FA_LIB_PATH=$L python tools/perf_probe.py decode 2>&1 | grep C5
done; done

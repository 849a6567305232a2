#!/bin/bash
# time the step kernels with each experiment build of the library (ADS_B200_LIB)
for lib in paper_1911_08158_b200/libads_b200.so paper_1911_08158_b200/libads_ablate_*.so; do
  echo "== $lib"; ADS_B200_LIB=$PWD/$lib timeout 200 python scripts/time_ops.py 2>&1 | grep "n=515"
done

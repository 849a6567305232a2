#!/bin/bash
# operator-kernel ablations (results are wrong; timing only): time kop at c4 with each
# libads_ablate_*.so built by scripts/build_ablate.py
for r in 1; do
for lib in paper_1911_08158_b200/libads_b200.so paper_1911_08158_b200/libads_ablate_*.so; do
  echo "== $lib"; ADS_B200_LIB=$PWD/$lib timeout 200 python scripts/time_kernels.py c4 2>&1 | tail -1
done; done

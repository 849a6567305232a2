#!/bin/bash
# A/B of library variants (ADS_B200_LIB): the main build and every libads_ablate_*.so, twice in
# alternating order, with the SM clock / power / throttle state after each run
for r in 1 2; do
for lib in paper_1911_08158_b200/libads_b200.so paper_1911_08158_b200/libads_ablate_*.so; do
  echo "== $lib"; ADS_B200_LIB=$PWD/$lib timeout 200 python scripts/time_ops.py 2>&1 | grep "n=515"
  nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_throttle_reasons.active --format=csv,noheader
done; done

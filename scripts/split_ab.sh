#!/bin/bash
# A/B of the split operator step (ADS_SPLIT=1) against the fused operator (ADS_SPLIT=0) -- a record of the
# reverted round-1 experiment; the current library has no split path and ignores ADS_SPLIT
for sp in 1 0 1; do echo "== ADS_SPLIT=$sp"; ADS_SPLIT=$sp timeout 300 python scripts/time_ops.py 2>&1 | grep -E "n=515|n=258 p=2"; ADS_SPLIT=$sp timeout 300 python scripts/time_configs.py 2>&1 | grep -E "c3|c4"; done

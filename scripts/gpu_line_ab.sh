# line-sweep A/B: parity suites, then slab and config timings with ADS_LINE_SWEEP=1 (default) and 0
timeout 1200 python -m pytest tests/test_gpu_slabs.py tests/test_gpu_parity.py tests/test_gpu_elastic.py -q -x -k "not full_size and not largest and not maximum" 2>&1 | tail -4
for v in 1 0; do echo "== ADS_LINE_SWEEP=$v"; ADS_LINE_SWEEP=$v timeout 300 python scripts/time_slabs.py c4 2>&1 | grep -v "all-to-all"; ADS_LINE_SWEEP=$v timeout 300 python scripts/time_configs.py 2>&1 | tail -6; done

timeout 900 python -m pytest tests/test_gpu_slabs.py -q -x > gpurun_out/r2_line_tests.log 2>&1; tail -2 gpurun_out/r2_line_tests.log
for v in 1 0; do echo "== ADS_LINE_SMEM=$v"; ADS_LINE_SMEM=$v timeout 300 python scripts/prof_slab_classes.py 4 8 2>&1 | sed 's/(launches.*//'; ADS_LINE_SMEM=$v timeout 300 python scripts/time_slabs.py c4 2>&1 | head -4; done

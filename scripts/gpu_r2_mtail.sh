timeout 1200 python -m pytest tests/test_gpu_modal.py -q -x > gpurun_out/r2_mtail_tests.log 2>&1; tail -2 gpurun_out/r2_mtail_tests.log
for v in 1 0; do echo "== ADS_MODAL_FUSE_TAIL=$v"; ADS_MODAL_FUSE_TAIL=$v timeout 300 python scripts/time_modal.py 2>&1 | head -8; done

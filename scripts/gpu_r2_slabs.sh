timeout 1500 python -m pytest tests/test_gpu_slabs.py -q -x 2>&1 | tail -3 > gpurun_out/r2_slab_tests.log
timeout 600 python scripts/time_slabs.py c4 > gpurun_out/r2_time_slabs.log 2>&1
cat gpurun_out/r2_slab_tests.log gpurun_out/r2_time_slabs.log

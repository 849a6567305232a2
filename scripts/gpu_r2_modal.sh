timeout 600 python scripts/time_modal.py c4 > gpurun_out/r2_time_modal.log 2>&1
timeout 900 python -m pytest tests/test_gpu_modal.py tests/test_gpu_parity.py -q -x -k "modal" 2>&1 | tail -5 > gpurun_out/r2_modal_tests.log
cat gpurun_out/r2_modal_tests.log gpurun_out/r2_time_modal.log

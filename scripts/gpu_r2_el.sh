timeout 1200 python -m pytest tests/test_gpu_elastic.py tests/test_gpu_parity.py -q -x -k "elastic or next_row" 2>&1 | tail -5 > gpurun_out/r2_el_tests.log
cat gpurun_out/r2_el_tests.log

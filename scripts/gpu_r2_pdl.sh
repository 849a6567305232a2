timeout 1500 python -m pytest tests/test_gpu_elastic.py tests/test_gpu_parity.py -q -x -k "not full_size" > gpurun_out/r2_pdl_tests.log 2>&1; tail -2 gpurun_out/r2_pdl_tests.log
for v in 1 0; do echo "== ADS_PDL=$v"; ADS_PDL=$v timeout 300 python scripts/time_configs.py 2>&1 | head -5; done

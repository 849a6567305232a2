timeout 900 python -m pytest tests/test_gpu_elastic.py -q -x -k "not full_size" > gpurun_out/r2_kron_tests.log 2>&1; tail -3 gpurun_out/r2_kron_tests.log
timeout 300 python scripts/time_c5.py 2>&1 | head -1
timeout 900 python scripts/time_elastic_scaled.py 256 512 > gpurun_out/r2_kron_scaled.log 2>&1; cat gpurun_out/r2_kron_scaled.log
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2_c5x512_launches_v2.csv python scripts/prof_c5_scaled.py 512 > gpurun_out/ncu_c5x512.log 2>&1

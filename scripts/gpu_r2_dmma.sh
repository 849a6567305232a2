# kop4 with the DMMA stage C: kernel times, then the non-slow GPU suite
timeout 300 python scripts/time_kernels.py c4 c3 c2 > gpurun_out/r2_time_dmma.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x -k "not slow" 2>&1 | tail -15 > gpurun_out/r2_t_dmma.log
cat gpurun_out/r2_time_dmma.log gpurun_out/r2_t_dmma.log

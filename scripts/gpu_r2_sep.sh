timeout 300 python scripts/time_setstate.py c4 > gpurun_out/r2_setstate.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x -k "not slow" 2>&1 | tail -3 > gpurun_out/r2_t_sep.log
cat gpurun_out/r2_setstate.log gpurun_out/r2_t_sep.log

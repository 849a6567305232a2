set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q -k "unit_operators or c1_full or c2_full or c3_recipe or c4_recipe or 2d_scheme or virtual_slabs_c4 or elastic_unit or c5_recipe" 2>&1 | tail -15 > gpurun_out/r2_t1.log
timeout 300 python scripts/time_kernels.py c4 c3 c2 > gpurun_out/r2_time_v4.log 2>&1
ADS_KOP_V3=1 timeout 300 python scripts/time_kernels.py c4 c3 c2 > gpurun_out/r2_time_v3.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "c4_full_size" 2>&1 | tail -15 > gpurun_out/r2_t2.log
cat gpurun_out/r2_t1.log gpurun_out/r2_time_v4.log gpurun_out/r2_time_v3.log gpurun_out/r2_t2.log

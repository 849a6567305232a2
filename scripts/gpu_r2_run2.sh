timeout 900 python -m pytest tests -m gpu -x -q -k "c4_full_size or unit_operators or c1_full or c2_full or c3_recipe or c4_recipe or 2d_scheme or virtual_slabs_c4 or elastic_unit or c5_recipe or other_degrees or largest_line or bitwise" 2>&1 | tail -5 > gpurun_out/r2_t1.log
timeout 300 python scripts/time_kernels.py c4 c3 c2 > gpurun_out/r2_time_v4.log 2>&1
cat gpurun_out/r2_t1.log gpurun_out/r2_time_v4.log

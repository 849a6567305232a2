# kop iteration: quick parity of the operator paths, then per-kernel times at c3/c4 and c5
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "unit_operators or c1_full or c2_full or c3_recipe or c4_recipe or anisotropic or kop_z_split or 2d_scheme or c4_full_size or other_degrees or bitwise" 2>&1 | tail -4
timeout 600 python -m pytest tests/test_gpu_slabs.py tests/test_gpu_elastic.py -q -x -k "not full_size" 2>&1 | tail -3
timeout 300 python scripts/time_kernels.py c3 c4

# quick check: slab + elastic + operator parity, then c5 / slab / config timings
timeout 900 python -m pytest tests/test_gpu_slabs.py tests/test_gpu_elastic.py tests/test_gpu_parity.py -q -x -k "not full_size and not largest and not maximum" 2>&1 | tail -2
timeout 120 python scripts/time_c5.py 2>&1 | head -1
timeout 300 python scripts/time_slabs.py c4 2>&1 | grep -v all-to-all
timeout 300 python scripts/time_configs.py 2>&1 | tail -5

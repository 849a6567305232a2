# c5 step time vs the z-piece counts of the kron3 / operator kernels, and the slab timings
timeout 600 python -m pytest tests/test_gpu_slabs.py -q -x 2>&1 | tail -2
for kz in 0 4 5 6 8 12 16; do for oz in 0 6; do echo -n "KRON_NZ=$kz KOP_NZ=$oz  "; ADS_KRON_NZ=$kz ADS_KOP_NZ=$oz timeout 120 python scripts/time_c5.py 2>&1 | head -1; done; done
timeout 300 python scripts/time_slabs.py c4 2>&1 | grep -v all-to-all

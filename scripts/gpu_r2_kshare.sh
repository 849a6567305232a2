timeout 900 python -m pytest tests/test_gpu_elastic.py -q -x > gpurun_out/r2_kshare_tests.log 2>&1; tail -2 gpurun_out/r2_kshare_tests.log
for v in 1 0; do echo "== ADS_KRON_SHARE=$v"; ADS_KRON_SHARE=$v timeout 300 python scripts/time_c5.py 2>&1 | head -1
  ADS_KRON_SHARE=$v timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ks_$v.csv python scripts/prof_c5_scaled.py 512 > /dev/null 2>&1
  python scripts/launch_agg.py gpurun_out/ks_$v.csv 37 2>&1 | head -6; done
ADS_KRON_SHARE=1 timeout 600 python scripts/time_elastic_scaled.py 256 > gpurun_out/r2_kshare_256.log 2>&1; cat gpurun_out/r2_kshare_256.log

for lib in paper_1911_08158_b200/libads_b200.so paper_1911_08158_b200/libads_ablate_ry2.so; do
  echo "== $lib"
  ADS_B200_LIB=$PWD/$lib timeout 300 python -m pytest tests/test_gpu_elastic.py -q -x -k "unit_operators" 2>&1 | tail -1
  ADS_B200_LIB=$PWD/$lib timeout 300 python scripts/time_c5.py 2>&1 | head -1
  ADS_B200_LIB=$PWD/$lib timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ry_$(basename $lib .so).csv python scripts/prof_c5_scaled.py 512 > /dev/null 2>&1
  python scripts/launch_agg.py gpurun_out/ry_$(basename $lib .so).csv 37 > gpurun_out/ry_$(basename $lib .so).txt; head -8 gpurun_out/ry_$(basename $lib .so).txt
done

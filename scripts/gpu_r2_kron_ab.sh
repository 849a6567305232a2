for lib in paper_1911_08158_b200/libads_b200.so paper_1911_08158_b200/libads_ablate_*.so; do
  echo "== $lib"
  ADS_B200_LIB=$PWD/$lib timeout 300 python scripts/time_c5.py 2>&1 | head -1
  ADS_B200_LIB=$PWD/$lib timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ab_$(basename $lib .so).csv python scripts/prof_c5_scaled.py 512 > /dev/null 2>&1
  python scripts/launch_agg.py gpurun_out/ab_$(basename $lib .so).csv 37 | head -5
done

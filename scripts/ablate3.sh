for lib in paper_1911_08158_b200/libads_b200.so paper_1911_08158_b200/libads_ablate_head.so paper_1911_08158_b200/libads_b200.so; do
  echo "== $lib"; ADS_B200_LIB=$PWD/$lib timeout 200 python scripts/time_ops.py 2>&1 | grep -E "n=515|n=258 p=2"
  ADS_B200_LIB=$PWD/$lib timeout 200 python scripts/time_2d.py 2>&1 | tail -2
done

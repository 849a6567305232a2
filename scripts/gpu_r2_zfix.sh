for lib in paper_1911_08158_b200/libads_b200.so paper_1911_08158_b200/libads_ablate_*.so; do
  echo "== $lib"; ADS_B200_LIB=$PWD/$lib timeout 300 python scripts/prof_slab_classes.py 2 8 2>&1 | tail -2
done

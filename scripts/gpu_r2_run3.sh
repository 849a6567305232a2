bash scripts/gpu_r2_run2.sh
bash scripts/gpu_r2_ncu_kop.sh

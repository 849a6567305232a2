# ncu full capture of the operator kernel at c4 (one launch after set_state's)
python scripts/prof_step.py c4 2 > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:kop4 -s 1 -c 1 -o gpurun_out/r2_kop4_dmma -f python scripts/prof_step.py c4 2 > gpurun_out/ncu_kop4.log 2>&1
tail -3 gpurun_out/ncu_kop4.log

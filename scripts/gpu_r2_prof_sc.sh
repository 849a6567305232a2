# launch lists: c4 as 8 virtual slabs (one step after warm-up) and c5 (two steps)
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_slabs8_launches.csv python scripts/prof_slabs.py 8 > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_c5_launches.csv python scripts/prof_c5.py > /dev/null 2>&1
ls -la gpurun_out/*.csv

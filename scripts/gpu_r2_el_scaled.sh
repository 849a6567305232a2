# f1 evidence: c5 recipe at 128/256/512^3 (timings, invariant, 256^3 one step vs the truth oracle),
# and the ncu launch list of one c5 step (direct launches)
python -c "import torch; print(torch.cuda.get_device_name(0))"
timeout 1500 python scripts/time_elastic_scaled.py 128 256 512 > gpurun_out/r2_el_scaled.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_c5_launches.csv python scripts/prof_c5.py > gpurun_out/r2_c5_ncu.log 2>&1
cat gpurun_out/r2_el_scaled.log

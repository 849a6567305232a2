# ncu --set full of the three sweeps of one c4 step; compute-sanitizer memcheck of the smoke run
python scripts/prof_step.py c4 1 > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 3 -c 3 -o gpurun_out/r2_sweeps -f python scripts/prof_step.py c4 1 > gpurun_out/ncu_sweeps.log 2>&1
tail -2 gpurun_out/ncu_sweeps.log
timeout 600 compute-sanitizer --tool memcheck --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_memcheck.log 2>&1; echo "memcheck rc=$?" >> gpurun_out/r2_memcheck.log
tail -5 gpurun_out/r2_memcheck.log

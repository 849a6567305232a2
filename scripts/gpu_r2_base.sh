# round-2 re-entry baseline: GPU suite, bench, launch list, ncu full of the operator kernel
timeout 2400 python -m pytest tests -m gpu -q -x 2>&1 | tail -25 > gpurun_out/r2b_pytest_gpu.log
timeout 900 python bench.py > gpurun_out/r2b_bench.json 2> gpurun_out/r2b_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2b_launches.csv python bench.py --steps 2 --warmup 3 --no-configs --no-cpu-baseline > gpurun_out/r2b_ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:kop4 -s 1 -c 1 -o gpurun_out/r2b_kop4 -f python scripts/prof_step.py c4 2 > gpurun_out/r2b_ncu_kop4.log 2>&1
tail -5 gpurun_out/r2b_pytest_gpu.log; tail -c 1500 gpurun_out/r2b_bench.json

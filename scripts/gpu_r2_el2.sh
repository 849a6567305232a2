timeout 1200 python -m pytest tests/test_gpu_elastic.py -q -x 2>&1 | tail -3 > gpurun_out/r2_el_tests.log
timeout 600 python bench.py --config c5 --steps 50 --warmup 5 --no-cpu-baseline --no-configs > gpurun_out/r2_bench_c5.json 2> gpurun_out/r2_bench_c5.err
cat gpurun_out/r2_el_tests.log; tail -c 1500 gpurun_out/r2_bench_c5.json; tail -3 gpurun_out/r2_bench_c5.err

# full GPU suite + bench (one call); logs under gpurun_out/
timeout 3000 python -m pytest tests -m gpu -q -x 2>&1 | tail -25 > gpurun_out/r2_pytest_gpu.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err
tail -25 gpurun_out/r2_pytest_gpu.log; tail -c 3000 gpurun_out/r2_bench.json; tail -5 gpurun_out/r2_bench.err

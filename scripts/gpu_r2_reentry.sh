# re-entry check of a freshly built tree: smoke, the full GPU suite, the default bench
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_re.log 2>&1; echo smoke rc=$? >> gpurun_out/smoke_re.log
timeout 900 python bench.py > gpurun_out/bench_re.json 2> gpurun_out/bench_re.err
timeout 2000 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_re.txt 2>&1; echo rc=$? >> gpurun_out/pytest_gpu_re.txt
tail -2 gpurun_out/smoke_re.log; tail -3 gpurun_out/pytest_gpu_re.txt; head -c 600 gpurun_out/bench_re.json

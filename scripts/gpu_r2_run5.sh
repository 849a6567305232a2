timeout 1500 python -m pytest tests -m gpu -q -x -k "not slow" 2>&1 | tail -3 > gpurun_out/r2_t5.log
timeout 300 python scripts/time_setstate.py c4 > gpurun_out/r2_setstate.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 --no-configs --no-cpu-baseline > gpurun_out/r2_bench_q.json 2>gpurun_out/r2_bench_q.err
cat gpurun_out/r2_t5.log gpurun_out/r2_setstate.log; python -c "
import json; d=json.loads(open('gpurun_out/r2_bench_q.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['e2e']['value'], {k:round(v['ms_per_launch'],4) for k,v in d['kernels'].items()})"

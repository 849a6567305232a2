#!/bin/bash
# One GPU call that refreshes the committed evidence for the current build (TAG names the version):
# ncu --set full capture of one step (kop + 3 sweeps), DRAM traffic JSON, bench (both arms),
# ncu launch list of a short bench, smoke, GPU tests.  Outputs land in gpurun_out/.
set -x
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"kop|sweep" -s 4 -c 4 -o gpurun_out/prof_r1_${TAG:-v6} python scripts/prof_step.py c4 2 > gpurun_out/ncu_full_${TAG:-v6}.log 2>&1
python scripts/ncu_traffic.py gpurun_out/prof_r1_${TAG:-v6}.ncu-rep gpurun_out/r1_${TAG:-v6}_traffic.json > /dev/null 2>&1 && cp gpurun_out/r1_${TAG:-v6}_traffic.json profiles/
timeout 600 python bench.py > gpurun_out/bench_${TAG:-v6}.json 2> gpurun_out/bench_${TAG:-v6}.err
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref_${TAG:-v6}.json 2> gpurun_out/bench_ref_${TAG:-v6}.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_${TAG:-v6}.csv python bench.py --steps 2 --warmup 3 > gpurun_out/ncu_launch_${TAG:-v6}.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${TAG:-v6}.log 2>&1; echo smoke rc=$? >> gpurun_out/smoke_${TAG:-v6}.log
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_${TAG:-v6}.txt 2>&1; echo rc=$? >> gpurun_out/pytest_gpu_${TAG:-v6}.txt

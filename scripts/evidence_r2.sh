#!/bin/bash
# Round-2 evidence for the current build (TAG names it): ncu --set full of the c4 operator kernel
# and its DRAM traffic, bench (c4 and c5, both arms), ncu launch list of a short bench,
# smoke, the full GPU suite, per-config / slab / set-state / modal timings.  Outputs in gpurun_out/.
T=${TAG:-r2_v1}
# (one kernel per capture: gpurun_out/ must stay under 64 MiB to come back)
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"kop" -s 1 -c 1 -o gpurun_out/prof_$T -f python scripts/prof_step.py c4 2 > gpurun_out/ncu_full_$T.log 2>&1
python scripts/ncu_traffic.py gpurun_out/prof_$T.ncu-rep gpurun_out/${T}_traffic.json > /dev/null 2>&1 && cp gpurun_out/${T}_traffic.json profiles/
timeout 900 python bench.py > gpurun_out/bench_$T.json 2> gpurun_out/bench_$T.err
timeout 600 python bench.py --config c5 --steps 50 --no-configs > gpurun_out/bench_c5_$T.json 2> gpurun_out/bench_c5_$T.err
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref_$T.json 2> gpurun_out/bench_ref_$T.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$T.csv python bench.py --steps 2 --warmup 3 --no-configs --no-cpu-baseline --repeats 1 > gpurun_out/ncu_launch_$T.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$T.log 2>&1; echo smoke rc=$? >> gpurun_out/smoke_$T.log
timeout 300 python scripts/time_configs.py > gpurun_out/configs_$T.log 2>&1
timeout 300 python scripts/time_kernels.py c3 c4 > gpurun_out/kernels_$T.log 2>&1
timeout 300 python scripts/time_slabs.py c4 > gpurun_out/slabs_$T.log 2>&1
timeout 300 python scripts/time_setstate.py c4 > gpurun_out/setstate_$T.log 2>&1
timeout 300 python scripts/time_modal.py > gpurun_out/modal_$T.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:kron3_kernel -s 14 -c 1 -o gpurun_out/kron3_$T -f python scripts/prof_c5_scaled.py 256 > gpurun_out/ncu_kron3_$T.log 2>&1
timeout 900 python scripts/time_elastic_scaled.py 128 256 512 > gpurun_out/el_scaled_$T.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/c5x512_launches_$T.csv python scripts/prof_c5_scaled.py 512 > /dev/null 2>&1
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_$T.txt 2>&1; echo rc=$? >> gpurun_out/pytest_gpu_$T.txt
# summaries on the box; the full reports stay there (gpurun_out/ must stay under 64 MiB)
python scripts/ncu_summary.py gpurun_out/prof_$T.ncu-rep > gpurun_out/ncu_summary_kop_$T.md 2>&1
python scripts/ncu_lines.py gpurun_out/prof_$T.ncu-rep kop4_kernelILi3 30 > gpurun_out/ncu_lines_kop_$T.txt 2>&1
python scripts/ncu_summary.py gpurun_out/kron3_$T.ncu-rep > gpurun_out/ncu_summary_kron3_$T.md 2>&1
python scripts/ncu_lines.py gpurun_out/kron3_$T.ncu-rep kron3_kernelILi2ELi2E 30 > gpurun_out/ncu_lines_kron3_$T.txt 2>&1
python scripts/launch_agg.py gpurun_out/c5x512_launches_$T.csv 37 > gpurun_out/c5x512_table_$T.txt 2>&1
rm -f gpurun_out/*.ncu-rep gpurun_out/c5x512_launches_$T.csv
du -sh gpurun_out
tail -3 gpurun_out/pytest_gpu_$T.txt; tail -2 gpurun_out/smoke_$T.log; cat gpurun_out/configs_$T.log gpurun_out/kernels_$T.log

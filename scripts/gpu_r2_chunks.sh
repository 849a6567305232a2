# chunk-pipelined single-GPU step: timings and bitwise equality at c4 / c3, quick parity with chunks
timeout 600 python scripts/time_chunks.py c4 1 2 3 4 6 8 > gpurun_out/r2_chunks_c4.log 2>&1
timeout 300 python scripts/time_chunks.py c3 1 2 4 8 > gpurun_out/r2_chunks_c3.log 2>&1
ADS_STEP_CHUNKS=4 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "c1_full or c2_full or c3_recipe or anisotropic or other_degrees" > gpurun_out/r2_chunks_pytest.log 2>&1
cat gpurun_out/r2_chunks_c4.log gpurun_out/r2_chunks_c3.log; tail -3 gpurun_out/r2_chunks_pytest.log

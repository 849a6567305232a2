# the multi-rank NCCL test file on this box (world 1 runs; 2 and 4 skip on a one-GPU box)
timeout 900 python -m pytest tests/test_gpu_nccl_multirank.py -m gpu -q -rs > gpurun_out/nccl_multirank.txt 2>&1; echo rc=$? >> gpurun_out/nccl_multirank.txt
cat gpurun_out/nccl_multirank.txt | tail -8

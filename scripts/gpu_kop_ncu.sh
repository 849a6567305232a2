# ncu --set full of one c4 operator-kernel launch (TAG names the capture)
python scripts/prof_step.py c4 2 > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:kop4 -s 1 -c 1 -o gpurun_out/${TAG} -f python scripts/prof_step.py c4 2 > gpurun_out/ncu_${TAG}.log 2>&1
tail -2 gpurun_out/ncu_${TAG}.log

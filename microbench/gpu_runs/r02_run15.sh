timeout 60 python microbench/time_kernels.py --config 5 --q 1 --reps 1 > gpurun_out/plain15.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k3_contract|k4_multi" -s 4 -c 2 -o gpurun_out/k3q1_k4 python microbench/time_kernels.py --config 5 --q 1 --reps 1 > gpurun_out/ncu15.log 2>&1
echo done $?

timeout 60 python microbench/time_kernels.py --config 5 --reps 3 > gpurun_out/plain13.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k5g_wgemm -s 2 -c 1 -o gpurun_out/k5g_v21 python microbench/time_kernels.py --config 5 --reps 1 > gpurun_out/ncu13.log 2>&1
echo done $?
cat gpurun_out/plain13.log

# K5g source-level warp-stall capture (cfg5, q = 2)
timeout 60 python microbench/time_kernels.py --config 5 --reps 1 > gpurun_out/plain22.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k5g_wgemm -s 2 -c 1 -o gpurun_out/k5g_src22 python microbench/time_kernels.py --config 5 --reps 1 > gpurun_out/ncu22.log 2>&1
echo done $?; tail -3 gpurun_out/ncu22.log

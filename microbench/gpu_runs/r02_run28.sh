# K2 and K5b full captures with source (cfg5)
timeout 60 python microbench/time_kernels.py --config 5 --reps 1 > gpurun_out/plain28.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k2_interpolate|k5b_reverse" -s 2 -c 2 -o gpurun_out/k2k5b_28 python microbench/time_kernels.py --config 5 --reps 1 > gpurun_out/ncu28.log 2>&1
echo done $?; tail -2 gpurun_out/ncu28.log

export IGA_LIB=microbench/libiga_IGA_EXPERIMENT_K3P.so
timeout 60 python microbench/time_kernels.py --config 5 --q 1 --reps 1 > gpurun_out/plain16.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k3p_contract" -s 2 -c 1 -o gpurun_out/k3p_q1 python microbench/time_kernels.py --config 5 --q 1 --reps 1 > gpurun_out/ncu16.log 2>&1
echo done $?

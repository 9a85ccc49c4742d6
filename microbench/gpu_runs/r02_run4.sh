IGA_LIB=microbench/libiga_IGA_EXPERIMENT_K3P_NO_STORE.so python microbench/time_kernels.py --config 5 --reps 1 > gpurun_out/plain4.log 2>&1 && \
IGA_LIB=microbench/libiga_IGA_EXPERIMENT_K3P_NO_STORE.so ncu --set full --clock-control none --import-source on -k regex:k3p_contract -s 2 -c 1 -o gpurun_out/k3p_nostore python microbench/time_kernels.py --config 5 --reps 1 > gpurun_out/ncu4a.log 2>&1
python microbench/time_kernels.py --config 5 --reps 1 > gpurun_out/plain4b.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k3p_contract -s 2 -c 1 -o gpurun_out/k3p_v2 python microbench/time_kernels.py --config 5 --reps 1 > gpurun_out/ncu4b.log 2>&1
echo done

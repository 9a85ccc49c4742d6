# clustered K3 with 2 and 4 row blocks per cluster
for lib in microbench/libiga_IGA_EXPERIMENT_K3_CLUSTER_IGA_K3_CL2.so microbench/libiga_IGA_EXPERIMENT_K3_CLUSTER_IGA_K3_CL4.so; do
  for q in 1 2; do IGA_LIB=$lib timeout 120 python microbench/time_kernels.py --config 5 --q $q --reps 5; done
done > gpurun_out/t25.log 2>&1
cat gpurun_out/t25.log

# K5g bounds: generator FP64 arithmetic and table streaming removed (timing only)
for lib in paper_2107_09568_b200/libiga.so microbench/libiga_IGA_EXPERIMENT_K5G_NO_GEN_MATH.so microbench/libiga_IGA_EXPERIMENT_K5G_NO_TABLE_REFILL.so microbench/libiga_IGA_EXPERIMENT_K5G_NO_GEN_MATH_IGA_EXPERIMENT_K5G_NO_TABLE_REFILL.so; do
  IGA_LIB=$lib timeout 120 python microbench/time_kernels.py --config 5 --reps 5
done > gpurun_out/t23.log 2>&1
cat gpurun_out/t23.log

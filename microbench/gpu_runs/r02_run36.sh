# scheduling sensitivity: policy created inside coop (run33 build) vs hoisted (HEAD), v22 reference
for i in 1 2 3; do for lib in microbench/libiga_IGA_EXPERIMENT_K3_COOP_V22.so microbench/libiga_hoist.so paper_2107_09568_b200/libiga.so; do
  IGA_LIB=$lib timeout 120 python microbench/time_kernels.py --config 5 --reps 5 | cut -c1-90
done; done

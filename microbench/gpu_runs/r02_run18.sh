for lib in microbench/libiga_IGA_K3_MI1.so paper_2107_09568_b200/libiga.so; do
  IGA_LIB=$lib timeout 60 python microbench/time_kernels.py --config 5 --reps 5
  IGA_LIB=$lib timeout 60 python microbench/time_kernels.py --config 5 --q 1 --reps 5
  IGA_LIB=$lib timeout 60 python microbench/time_kernels.py --config 3 --q 1 --reps 5
done

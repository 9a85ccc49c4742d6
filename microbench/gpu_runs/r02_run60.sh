# pipelined K3 with the refill before the tail DMMAs; DMMA order ni-major variant
for lib in paper_2107_09568_b200/libiga.so microbench/libiga_IGA_EXPERIMENT_K3_NI_MAJOR.so; do
  echo $lib; IGA_LIB=$lib timeout 120 python microbench/time_kernels.py --config 5 --q 2 --reps 5 | cut -c1-100
done

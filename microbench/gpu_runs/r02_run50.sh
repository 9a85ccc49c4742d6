# full-sector stores for one pass only (timing only)
for lib in paper_2107_09568_b200/libiga.so microbench/libiga_IGA_EXPERIMENT_K3_FULLSECTOR1.so microbench/libiga_IGA_EXPERIMENT_K3_FULLSECTOR2.so; do
  for q in 1 2; do IGA_LIB=$lib timeout 120 python microbench/time_kernels.py --config 5 --q $q --reps 5 | cut -c1-90; done
done

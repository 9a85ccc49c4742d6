# apply epilogue, two-level run sums: cost of level 1 / level 2 / the extra barrier (timing only)
for lib in microbench/libiga_IGA_EXPERIMENT_APPLY_NO_L1.so microbench/libiga_IGA_EXPERIMENT_APPLY_NO_L2.so microbench/libiga_IGA_EXPERIMENT_APPLY_NO_L1_IGA_EXPERIMENT_APPLY_NO_L2.so; do
  echo $lib; IGA_LIB=$lib timeout 120 python microbench/time_kernels.py --config 5 --apply --reps 3 | grep -o '"apply": [0-9.]*'
done

# apply epilogue bounds (timing only, wrong y): no FP64 block products, no in-order run sums, neither
for lib in paper_2107_09568_b200/libiga.so microbench/libiga_IGA_EXPERIMENT_APPLY_NO_PROD.so microbench/libiga_IGA_EXPERIMENT_APPLY_NO_RUNSUM.so microbench/libiga_IGA_EXPERIMENT_APPLY_NO_PROD_IGA_EXPERIMENT_APPLY_NO_RUNSUM.so; do
  echo $lib; IGA_LIB=$lib timeout 120 python microbench/time_kernels.py --config 5 --apply --reps 3 | grep -o '"apply": [0-9.]*'
done

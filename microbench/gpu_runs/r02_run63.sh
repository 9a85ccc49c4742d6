# timing probe: part-2 chunks interleaved with part-1 chunks (wrong K), with and without the epilogue
for lib in microbench/libiga_IGA_EXPERIMENT_K3_INTERLEAVE.so microbench/libiga_IGA_EXPERIMENT_K3_INTERLEAVE_IGA_EXPERIMENT_K3_BARE.so microbench/libiga_IGA_EXPERIMENT_K3_BARE.so paper_2107_09568_b200/libiga.so; do
  echo $lib; IGA_LIB=$lib timeout 120 python microbench/time_kernels.py --config 5 --q 2 --reps 5 | grep -o '"K3": [0-9.]*'
done

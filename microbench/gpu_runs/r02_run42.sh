# K3 epilogue code-shape variants: tile-loop unroll 1 / 2, split passes
for i in 1 2; do for lib in paper_2107_09568_b200/libiga.so microbench/libiga_IGA_K3_TILE_UNROLL1.so microbench/libiga_IGA_K3_TILE_UNROLL2.so microbench/libiga_IGA_EXPERIMENT_K3_SPLIT_PASSES.so; do
  for q in 1 2; do IGA_LIB=$lib timeout 120 python microbench/time_kernels.py --config 5 --q $q --reps 5 | cut -c1-90; done
done; done

# K5g: 2 table stages with 10 / 12 X̃ stages vs (3, 8)
for i in 1 2; do for lib in paper_2107_09568_b200/libiga.so microbench/libiga_IGA_K5G_SA2_IGA_K5G_SB12.so microbench/libiga_IGA_K5G_SA2_IGA_K5G_SB10.so; do
  IGA_LIB=$lib timeout 120 python microbench/time_kernels.py --config 5 --reps 5 | cut -c1-120
done; done

# K5g ring shapes: (4,5), (4,4), (3,9) vs (3,8)
for i in 1 2; do for lib in paper_2107_09568_b200/libiga.so microbench/libiga_IGA_K5G_SA4_IGA_K5G_SB5.so microbench/libiga_IGA_K5G_SA4_IGA_K5G_SB4.so microbench/libiga_IGA_K5G_SA3_IGA_K5G_SB9.so; do
  IGA_LIB=$lib timeout 120 python microbench/time_kernels.py --config 5 --reps 5 | cut -c1-110
done; done

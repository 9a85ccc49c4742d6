# K3 with 2 ring stages and 5 CTAs per SM (94 registers, 37.4 KB shared memory per CTA)
for lib in paper_2107_09568_b200/libiga.so microbench/libiga_IGA_K3_STAGES2.so microbench/libiga_IGA_K3_STAGES2_IGA_K3_MINB5.so; do
  for q in 2 1; do echo "$lib q=$q"; IGA_LIB=$lib timeout 120 python microbench/time_kernels.py --config 5 --q $q --reps 5 | cut -c1-120; done
done

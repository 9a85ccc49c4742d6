# K4 as a persistent grid-stride kernel with the next chunk's descriptors prefetched: parity and timing
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "csr_values or symmetric or edge_case or sharded_assembly" 2>&1 | tail -2
for lib in paper_2107_09568_b200/libiga.so microbench/libiga_IGA_K4_MINB2.so microbench/libiga_IGA_K4_MINB2_IGA_K4_WAVES2.so microbench/libiga_IGA_EXPERIMENT_K4_NOLOOP.so; do
  echo $lib; IGA_LIB=$lib timeout 120 python microbench/time_kernels.py --config 5 --reps 5 | grep -o '"K4": [0-9.]*'
done

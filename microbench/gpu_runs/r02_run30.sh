# K4: both blocks' first two slots in one round trip (product) vs 64-register cap vs serial sums
for i in 1 2; do for lib in microbench/libiga_IGA_EXPERIMENT_K4_SERIAL_SUMS.so paper_2107_09568_b200/libiga.so microbench/libiga_IGA_K4_MINB4.so; do
  IGA_LIB=$lib timeout 120 python microbench/time_kernels.py --config 5 --reps 5 | cut -c1-110
done; done
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "csr_values or symmetric or sharded or edge_case or host_pointers" 2>&1 | tail -2

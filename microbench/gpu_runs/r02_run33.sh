# K3 cooperative store with per-lane precomputed shared-memory offsets vs v22
for i in 1 2; do for lib in microbench/libiga_IGA_EXPERIMENT_K3_COOP_V22.so paper_2107_09568_b200/libiga.so; do
  for q in 1 2; do IGA_LIB=$lib timeout 120 python microbench/time_kernels.py --config 5 --q $q --reps 5 | cut -c1-100; done
done; done
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "csr_values or symmetric or sharded or edge_case or host_pointers or nurbs" 2>&1 | tail -2

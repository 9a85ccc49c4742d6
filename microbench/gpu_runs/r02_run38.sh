# K3 epilogue map loads through one 16-B row descriptor (two load levels instead of three)
for i in 1 2; do for lib in paper_2107_09568_b200/libiga.so microbench/libiga_IGA_EXPERIMENT_K3_ROWDESC.so; do
  for q in 1 2; do IGA_LIB=$lib timeout 120 python microbench/time_kernels.py --config 5 --q $q --reps 5 | cut -c1-90; done
done; done
IGA_LIB=microbench/libiga_IGA_EXPERIMENT_K3_ROWDESC.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "csr_values or symmetric or sharded or edge_case" 2>&1 | tail -1

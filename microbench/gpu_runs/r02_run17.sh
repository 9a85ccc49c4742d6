for lib in microbench/libiga_IGA_EXPERIMENT_K3P.so paper_2107_09568_b200/libiga.so; do
  IGA_LIB=$lib timeout 60 python microbench/time_kernels.py --config 5 --reps 5
  IGA_LIB=$lib timeout 60 python microbench/time_kernels.py --config 5 --q 1 --reps 5
done
IGA_LIB=microbench/libiga_IGA_EXPERIMENT_K3P.so timeout 300 python -m pytest -x -q -m gpu tests/test_gpu_parity.py -k "csr_values or pattern or edge_case or sharded or symmetric" 2>&1 | tail -2

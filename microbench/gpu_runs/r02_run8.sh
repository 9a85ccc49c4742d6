for lib in paper_2107_09568_b200/libiga.so microbench/libiga_IGA_EXPERIMENT_K3P_NO_STORE.so; do
  IGA_LIB=$lib timeout 60 python microbench/time_kernels.py --config 5 --reps 5
  IGA_LIB=$lib timeout 60 python microbench/time_kernels.py --config 5 --q 1 --reps 5
  IGA_LIB=$lib timeout 60 python microbench/time_kernels.py --config 4 --reps 3
done > gpurun_out/tk7.log 2>&1
cat gpurun_out/tk7.log
timeout 300 python -m pytest -x -q -m gpu tests/test_gpu_parity.py -k "csr_values or pattern or edge_case or sharded or symmetric" 2>&1 | tail -2

# product (pass lambdas, handle lock) vs HEAD lib, and the concurrency test
for i in 1 2; do for lib in microbench/libiga_head.so paper_2107_09568_b200/libiga.so; do
  for q in 1 2; do IGA_LIB=$lib timeout 120 python microbench/time_kernels.py --config 5 --q $q --reps 5; done
done; done > gpurun_out/t26.log 2>&1
cat gpurun_out/t26.log | cut -c1-110
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "concurrent or csr_values or host_pointers or sharded" 2>&1 | tail -3

# nzdata epilogue: 16-B stores vs scalar
for i in 1 2; do for lib in microbench/libiga_prev_epi0.so paper_2107_09568_b200/libiga.so; do
  IGA_LIB=$lib timeout 120 python microbench/time_kernels.py --config 5 --reps 3 --local
done; done
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "element_matrix or edge_case" 2>&1 | tail -2

# K2 tile-fastest thread mapping: timing + parity
for i in 1 2; do for lib in microbench/libiga_head.so paper_2107_09568_b200/libiga.so; do
  IGA_LIB=$lib timeout 120 python microbench/time_kernels.py --config 5 --reps 5 | cut -c1-100
done; done
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_projection.py -x -q -m gpu 2>&1 | tail -2

# K5g DFMA tail groups (modes 13-16) vs none
for i in 1 2; do for lib in paper_2107_09568_b200/libiga.so microbench/libiga_IGA_EXPERIMENT_K5G_NO_TAIL.so; do
  for c in 5 3; do IGA_LIB=$lib timeout 120 python microbench/time_kernels.py --config $c --reps 5 | cut -c1-110; done
done; done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_projection.py tests/test_gpu_fullsize.py -x -q -m gpu -k "sensitivity or combined or nurbs or anisotropic or l2_projection" 2>&1 | tail -2

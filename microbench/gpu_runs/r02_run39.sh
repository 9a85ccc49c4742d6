# K5g with separate table / X̃ rings: (3 table, 8 X̃) product vs (3,6), (3,4) and the single 4-stage ring
for i in 1 2; do for lib in microbench/libiga_hoist.so paper_2107_09568_b200/libiga.so microbench/libiga_IGA_K5G_SB6.so microbench/libiga_IGA_K5G_SB4.so; do
  IGA_LIB=$lib timeout 120 python microbench/time_kernels.py --config 5 --reps 5 | cut -c1-120
done; done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_projection.py -x -q -m gpu -k "sensitivity or combined or nurbs or anisotropic or l2_projection" 2>&1 | tail -1

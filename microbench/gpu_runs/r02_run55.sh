# K4 v26 (16-B descriptor and slot loads) vs store hint / CTAs per SM
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1
for lib in paper_2107_09568_b200/libiga.so microbench/libiga_IGA_EXPERIMENT_K4_ST_HINT.so microbench/libiga_IGA_K4_MINB4.so microbench/libiga_IGA_K4_MINB2.so; do
  echo $lib; IGA_LIB=$lib timeout 120 python microbench/time_kernels.py --config 5 --q 2 --reps 5 | cut -c1-100
done

# apply epilogue with two-level run sums: parity (apply tests) and timing, group sizes 3/4/6/8
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "apply or edge_case" 2>&1 | tail -2
for lib in paper_2107_09568_b200/libiga.so microbench/libiga_IGA_APPLY_AG3.so microbench/libiga_IGA_APPLY_AG6.so microbench/libiga_IGA_APPLY_AG8.so; do
  echo $lib; IGA_LIB=$lib timeout 120 python microbench/time_kernels.py --config 5 --apply --reps 3 | grep -o '"apply": [0-9.]*'
done
timeout 120 python microbench/time_kernels.py --config 4 --apply --reps 3 | grep -o '"apply": [0-9.]*'

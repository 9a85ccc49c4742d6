# K3: coefficient chunks copied without their zero column tiles (L2 -> SM traffic -24%); plain loop and pipelined loop
for lib in paper_2107_09568_b200/libiga.so microbench/libiga_IGA_EXPERIMENT_K3_PIPE.so; do
  echo $lib; for q in 2 1; do IGA_LIB=$lib timeout 120 python microbench/time_kernels.py --config 5 --q $q --reps 5 | grep -o '"K3": [0-9.]*'; done
done
timeout 120 python microbench/time_kernels.py --config 4 --reps 5 | grep -o '"K3": [0-9.]*'
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2

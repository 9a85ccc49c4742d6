# K3 with thread-block clusters of 8 row blocks: pooled transposed pass
C=microbench/libiga_IGA_EXPERIMENT_K3_CLUSTER.so
for lib in paper_2107_09568_b200/libiga.so $C; do
  for q in 0 1 2; do IGA_LIB=$lib timeout 120 python microbench/time_kernels.py --config 5 --q $q --reps 5; done
done > gpurun_out/t24.log 2>&1
cat gpurun_out/t24.log
IGA_LIB=$C timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/p24.log 2>&1; echo "pytest rc=$?" >> gpurun_out/p24.log
tail -3 gpurun_out/p24.log
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_requests_srcunit_tex_op_write.sum,lts__t_sectors_srcunit_tex_op_write.sum,lts__d_sectors_fill_device.sum
for q in 1 2; do
  echo "== cluster q=$q"
  IGA_LIB=$C timeout 300 ncu --metrics $M --clock-control none -k regex:k3_contract -s 2 -c 1 --csv python microbench/time_kernels.py --config 5 --q $q --reps 1 2>/dev/null | grep 'k3_contract' | awk -F'","' '{print $(NF-2), $(NF-1), $NF}'
done > gpurun_out/n24.log 2>&1
cat gpurun_out/n24.log

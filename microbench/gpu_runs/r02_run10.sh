for lib in paper_2107_09568_b200/libiga.so microbench/libiga_IGA_EXPERIMENT_K3P_NO_STORE.so; do
  IGA_LIB=$lib timeout 60 python microbench/time_kernels.py --config 5 --reps 5
  IGA_LIB=$lib timeout 60 python microbench/time_kernels.py --config 5 --q 1 --reps 5
  IGA_LIB=$lib timeout 60 python microbench/time_kernels.py --config 4 --reps 3
done > gpurun_out/tk10.log 2>&1
cat gpurun_out/tk10.log
timeout 300 python -m pytest -x -q -m gpu tests/test_gpu_parity.py -k "csr_values or pattern or edge_case or sharded or symmetric" 2>&1 | tail -2
timeout 60 python microbench/time_kernels.py --config 5 --reps 1 > gpurun_out/plain10.log 2>&1 && \
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active,lts__t_sector_op_read_hit_rate.pct --clock-control none -k regex:k3p_contract -s 2 -c 1 --csv python microbench/time_kernels.py --config 5 --reps 1 > gpurun_out/ncu10.csv 2>&1
tail -8 gpurun_out/ncu10.csv

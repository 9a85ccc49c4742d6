# where the K3 scatter time goes: pass split, scatter addresses vs contiguous stores, q = 0/1/2
P=paper_2107_09568_b200/libiga.so
for lib in $P microbench/libiga_IGA_EXPERIMENT_K3_LINEAR.so microbench/libiga_IGA_EXPERIMENT_NO_PASS1.so microbench/libiga_IGA_EXPERIMENT_NO_PASS2.so microbench/libiga_IGA_EXPERIMENT_NO_SCATTER.so; do
  for q in 0 1 2; do IGA_LIB=$lib timeout 120 python microbench/time_kernels.py --config 5 --q $q --reps 5; done
done > gpurun_out/t21.log 2>&1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_requests_srcunit_tex_op_write.sum,lts__t_sectors_srcunit_tex_op_write.sum,lts__d_sectors_fill_device.sum,l1tex__t_requests_pipe_lsu_mem_global_op_st.sum,lts__t_sector_op_write_hit_rate.pct
for lib in $P microbench/libiga_IGA_EXPERIMENT_K3_LINEAR.so microbench/libiga_IGA_EXPERIMENT_NO_PASS2.so; do
  for q in 0 1; do
    echo "== $lib q=$q"
    IGA_LIB=$lib timeout 300 ncu --metrics $M --clock-control none -k regex:k3_contract -s 2 -c 1 --csv python microbench/time_kernels.py --config 5 --q $q --reps 1 2>/dev/null | grep 'k3_contract' | awk -F'","' '{print $(NF-2), $(NF-1), $NF}'
  done
done > gpurun_out/n21.log 2>&1
cat gpurun_out/t21.log gpurun_out/n21.log

M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_op_read_hit_rate.pct,lts__d_sectors_fill_device.sum
for lib in paper_2107_09568_b200/libiga.so microbench/libiga_IGA_EXPERIMENT_K3_TABLE_EVICT_LAST.so microbench/libiga_IGA_EXPERIMENT_K3_STORE_EVICT_FIRST.so microbench/libiga_IGA_EXPERIMENT_K3_TABLE_EVICT_LAST_IGA_EXPERIMENT_K3_STORE_EVICT_FIRST.so microbench/libiga_IGA_EXPERIMENT_NO_SCATTER.so; do
  for q in 2 1; do
    IGA_LIB=$lib timeout 60 python microbench/time_kernels.py --config 5 --q $q --reps 5
    IGA_LIB=$lib timeout 300 ncu --metrics $M --clock-control none -k regex:k3_contract -s 2 -c 1 --csv python microbench/time_kernels.py --config 5 --q $q --reps 1 2>/dev/null | grep '"k3_contract\|k3_contract' | awk -F'","' '{print $(NF-2), $NF}'
  done
done > gpurun_out/l2pol.log 2>&1
cat gpurun_out/l2pol.log

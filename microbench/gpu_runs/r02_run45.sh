# per-pass L2 store policies: timing and DRAM traffic of K3
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_requests_srcunit_tex_op_write.sum
for lib in paper_2107_09568_b200/libiga.so microbench/libiga_IGA_EXPERIMENT_K3_PASS2_EVICT_NORMAL.so microbench/libiga_IGA_EXPERIMENT_K3_PASS2_EVICT_LAST.so; do
  for q in 1 2; do
    IGA_LIB=$lib timeout 120 python microbench/time_kernels.py --config 5 --q $q --reps 5 | cut -c1-90
    IGA_LIB=$lib timeout 300 ncu --metrics $M --clock-control none -k regex:k3_contract -s 2 -c 1 --csv python microbench/time_kernels.py --config 5 --q $q --reps 1 2>/dev/null | grep 'k3_contract' | awk -F'","' '{print $(NF-2), $NF}' | tr '\n' ' '; echo
  done
done

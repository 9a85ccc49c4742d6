# pipelined K3: bare main loop A/B and a source-level capture of the product K3
for lib in microbench/libiga_IGA_EXPERIMENT_K3_BARE.so microbench/libiga_IGA_EXPERIMENT_K3_BARE_IGA_EXPERIMENT_K3_NOPIPE.so; do
  echo $lib; IGA_LIB=$lib timeout 120 python microbench/time_kernels.py --config 5 --q 2 --reps 5 | cut -c1-100
done
timeout 400 ncu --set full --clock-control none --import-source on -k regex:k3_contract -s 1 -c 1 -o gpurun_out/k3_pipe python microbench/time_kernels.py --config 5 --reps 1 > gpurun_out/ncu58.log 2>&1; echo ncu $?

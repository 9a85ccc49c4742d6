# K3 register-direct scatter vs the staged cooperative scatter
D=microbench/libiga_IGA_EXPERIMENT_K3_DIRECT.so
for lib in paper_2107_09568_b200/libiga.so $D; do
  for q in 2 1; do IGA_LIB=$lib timeout 120 python microbench/time_kernels.py --config 5 --q $q --reps 5; done
done > gpurun_out/t20.log 2>&1
IGA_LIB=$D timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/p20.log 2>&1; echo "pytest rc=$?" >> gpurun_out/p20.log
cat gpurun_out/t20.log; tail -3 gpurun_out/p20.log

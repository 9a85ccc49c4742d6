# K3 staging without the FP64 adds L+ +- L- (timing only): does DADD interleaved with DMMA cost?
for i in 1 2; do for lib in paper_2107_09568_b200/libiga.so microbench/libiga_IGA_EXPERIMENT_K3_NO_STAGE_DADD.so; do
  IGA_LIB=$lib timeout 120 python microbench/time_kernels.py --config 5 --reps 5 --local | cut -c1-200
done; done

# pipelined K3, nmi==2 warps only in the pipelined loop (no spills): timing first, then parity
for lib in paper_2107_09568_b200/libiga.so microbench/libiga_IGA_EXPERIMENT_K3_BARE.so; do
  echo $lib; IGA_LIB=$lib timeout 120 python microbench/time_kernels.py --config 5 --q 2 --reps 5 | cut -c1-100
done
timeout 120 python microbench/time_kernels.py --config 5 --q 1 --reps 5 | cut -c1-100
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2

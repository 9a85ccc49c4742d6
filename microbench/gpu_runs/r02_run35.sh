# bench-step K3 with the v22 coop vs the offset-precomputed coop (same box, alternating)
for i in 1 2; do for lib in microbench/libiga_IGA_EXPERIMENT_K3_COOP_V22.so paper_2107_09568_b200/libiga.so; do
  IGA_LIB=$lib python bench.py --no-cpu-baseline --no-e2e --steps 20 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$lib', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['kernel_ms_per_step'].items()})"
  IGA_LIB=$lib timeout 120 python microbench/time_kernels.py --config 5 --reps 5 | cut -c1-90
done; done

# K4 beside the sensitivity chain (high-priority stream) vs serial
for i in 1 2; do for lib in paper_2107_09568_b200/libiga.so microbench/libiga_IGA_EXPERIMENT_K4_OVERLAP.so; do
  IGA_LIB=$lib python bench.py --no-cpu-baseline --no-e2e --steps 20 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$lib', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['kernel_ms_per_step'].items()})"
done; done
IGA_LIB=microbench/libiga_IGA_EXPERIMENT_K4_OVERLAP.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "combined or host_pointers" 2>&1 | tail -1

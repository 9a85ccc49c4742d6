# K4: bulk-staged pass-1 slots without the CTA barrier wait on thread 0
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "assembl or scatter or K_values or full" 2>&1 | tail -2
for q in 2 1; do timeout 120 python microbench/time_kernels.py --config 5 --q $q --reps 5 | cut -c1-120; done

# K3 main loop software-pipelined across chunk boundaries (k3_fast_chunk): parity + timing
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3
for q in 2 1; do timeout 120 python microbench/time_kernels.py --config 5 --q $q --reps 5 | cut -c1-160; done
timeout 120 python microbench/time_kernels.py --config 4 --reps 5 | cut -c1-160

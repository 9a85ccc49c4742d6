# apply epilogue with warp-shuffle segmented run sums: parity and timing
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "apply or edge_case" 2>&1 | tail -2
for c in 5 4 3; do timeout 120 python microbench/time_kernels.py --config $c --apply --reps 3 | grep -o '"apply": [0-9.]*'; done

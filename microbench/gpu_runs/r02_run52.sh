# K4 with 16-B descriptors and 16-B slot loads (slot ranges start at even slots)
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3
for q in 2 1; do timeout 120 python microbench/time_kernels.py --config 5 --q $q --reps 5 | cut -c1-120; done
timeout 300 ncu --set full --clock-control none -k regex:k4_multi -s 1 -c 1 -o gpurun_out/k4_v26 python microbench/time_kernels.py --config 5 --reps 1 > gpurun_out/ncu52.log 2>&1; echo ncu $?

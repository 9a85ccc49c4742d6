# checkpoint v25: full GPU suite, bench lines, launch list, full capture of K3/K5g/K4
set -x
python -m pytest tests/ -x -q -m gpu --durations=10 > gpurun_out/pytest_gpu_v25.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_v25.log
python bench.py > gpurun_out/bench_v25.json 2> gpurun_out/bench_v25.err; echo "bench rc=$?"
python bench.py --select-degree 1e-3 --no-cpu-baseline > gpurun_out/bench_q65_v25.json 2> gpurun_out/bench_q65_v25.err
for c in 1 2 3 4; do python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_cfg${c}_v25.json 2> /dev/null; done
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_v25.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo "launch rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k3_contract|k5g_wgemm|k4_multi" -s 3 -c 3 -o gpurun_out/full_v25 python microbench/time_kernels.py --config 5 --reps 1 > gpurun_out/ncu_full_v25.log 2>&1; echo "full rc=$?"
ncu -i gpurun_out/full_v25.ncu-rep --page raw --csv > gpurun_out/full_v25_raw.csv 2>/dev/null
tail -2 gpurun_out/pytest_gpu_v25.log

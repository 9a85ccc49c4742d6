# round-2 checkpoint: full GPU suite, bench lines (BASELINE cfg5 and the Eq. 65 degree), launch list, full captures
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m pytest tests/ -x -q -m gpu --durations=15 > gpurun_out/pytest_gpu_r02b.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_r02b.log
python bench.py > gpurun_out/bench_r02b.json 2> gpurun_out/bench_r02b.err; echo "bench rc=$?"
python bench.py --select-degree 1e-3 --no-cpu-baseline > gpurun_out/bench_q65_r02b.json 2> gpurun_out/bench_q65_r02b.err; echo "bench q65 rc=$?"
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_r02b.json 2> gpurun_out/bench_ref_r02b.err; echo "ref rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r02b.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch_r02b.log 2>&1; echo "launch rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k3_contract|k5g_wgemm|k4_multi" -s 3 -c 3 -o gpurun_out/full_r02b python microbench/time_kernels.py --config 5 --reps 1 > gpurun_out/ncu_full_r02b.log 2>&1; echo "full rc=$?"
ncu -i gpurun_out/full_r02b.ncu-rep --page raw --csv > gpurun_out/full_r02b_raw.csv 2>/dev/null
tail -3 gpurun_out/pytest_gpu_r02b.log; cat gpurun_out/bench_r02b.json | cut -c1-300

# Round-2 v26 checkpoint at HEAD (re-created container): full GPU suite, smoke, bench lines, launch list, full capture
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_v26.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu_v26.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
python bench.py > gpurun_out/bench_v26.json 2> gpurun_out/bench_v26.err; echo "bench rc=$?"
python bench.py --select-degree 1e-3 --no-cpu-baseline > gpurun_out/bench_q65_v26.json 2> gpurun_out/bench_q65_v26.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_v26.json 2>/dev/null
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_v26.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo "launch rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k3_contract|k5g_wgemm|k4_multi|k2_interpolate|k5b' -s 6 -c 6 -o gpurun_out/full_v26 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full_v26.log 2>&1; echo "full rc=$?"
cut -c1-400 gpurun_out/bench_v26.json

# Round-2 v27 checkpoint (v26 kernels + the shuffle-sum apply epilogue): full GPU suite, smoke, bench lines, launch list
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_v27.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu_v27.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python bench.py > gpurun_out/bench_v27.json 2> gpurun_out/bench_v27.err; echo "bench rc=$?"
python bench.py --select-degree 1e-3 --no-cpu-baseline > gpurun_out/bench_q65_v27.json 2> gpurun_out/bench_q65_v27.err
for c in 1 2 3 4; do python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_cfg${c}_v27.json 2> /dev/null; done
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_v27.json 2>/dev/null
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_v27.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo "launch rc=$?"
python -c "import json; d=json.load(open('gpurun_out/bench_v27.json')); print(d['ms_per_step'], {k: round(v['ms_median'],3) for k,v in d['windows'].items() if isinstance(v, dict)})"

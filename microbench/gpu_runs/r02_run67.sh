# bench with the matrix_free_apply window (compute-sanitizer is closed on this pool: not run)
python bench.py --no-cpu-baseline > gpurun_out/bench_v26c.json 2> gpurun_out/bench_v26c.err; echo "bench rc=$?"
python -c "import json; d=json.load(open('gpurun_out/bench_v26c.json')); print({k: round(v['ms_median'],3) for k,v in d['windows'].items() if isinstance(v, dict)})"

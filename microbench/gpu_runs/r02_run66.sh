# HEAD validation after the K3 experiment flags were added (product SASS of K3 unchanged): full GPU suite, smoke, bench
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_v26b.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu_v26b.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python bench.py --no-cpu-baseline > gpurun_out/bench_v26b.json 2> gpurun_out/bench_v26b.err; echo "bench rc=$?"
cut -c1-330 gpurun_out/bench_v26b.json

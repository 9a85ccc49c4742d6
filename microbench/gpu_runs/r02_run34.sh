# bench lines, v24 kernels (coop offsets, K4 descriptors, nzdata 16-B stores, K2 tile-fastest)
python bench.py > gpurun_out/bench_v24.json 2> gpurun_out/bench_v24.err; echo "bench rc=$?"
python bench.py --select-degree 1e-3 --no-cpu-baseline > gpurun_out/bench_q65_v24.json 2> gpurun_out/bench_q65_v24.err; echo "q65 rc=$?"
for c in 1 2 3 4; do python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_cfg${c}_v24.json 2> gpurun_out/bench_cfg${c}_v24.err; echo "cfg$c rc=$?"; done

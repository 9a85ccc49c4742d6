set -x
python -m pytest -x -q -m gpu tests/test_gpu_parity.py -k "csr_values or pattern or symmetric or sharded or edge_case or host_pointers or young or degenerate or nurbs or volume" > gpurun_out/pytest_quick.log 2>&1; echo "quick rc=$?"
tail -3 gpurun_out/pytest_quick.log
python -m pytest -x -q -m gpu tests/test_gpu_multiproc.py > gpurun_out/pytest_mp.log 2>&1; echo "mp rc=$?"
tail -3 gpurun_out/pytest_mp.log
for i in 1 2; do
IGA_LIB=microbench/libiga_IGA_EXPERIMENT_K3_CLASSIC.so python microbench/time_kernels.py --config 5 --reps 5
python microbench/time_kernels.py --config 5 --reps 5
done > gpurun_out/tk.log 2>&1
cat gpurun_out/tk.log
python microbench/time_kernels.py --config 5 --q 1 --reps 5 >> gpurun_out/tk.log 2>&1
IGA_LIB=microbench/libiga_IGA_EXPERIMENT_K3_CLASSIC.so python microbench/time_kernels.py --config 5 --q 1 --reps 5 >> gpurun_out/tk.log 2>&1
python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
python microbench/time_kernels.py --config 5 --reps 1 > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k3p_contract -s 2 -c 1 -o gpurun_out/k3p_full python microbench/time_kernels.py --config 5 --reps 1 > gpurun_out/ncu_full.log 2>&1; echo "ncu rc=$?"

# FP64 stores in runs of R doubles at random positions (the CSR scatter's store pattern)
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gpurun_out/store_runs microbench/store_runs.cu && ./gpurun_out/store_runs > gpurun_out/store_runs.jsonl 2>&1
cat gpurun_out/store_runs.jsonl
rm -f gpurun_out/store_runs

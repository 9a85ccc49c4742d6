# full capture of the apply-epilogue K3 (second k3_contract launch of time_kernels --apply)
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k3_contract -s 1 -c 1 -o gpurun_out/apply_k3 python microbench/time_kernels.py --config 5 --apply --reps 1 > gpurun_out/ncu65.log 2>&1; echo ncu $?

# full capture of the v27 apply path (u gather, K3 with the shuffle-sum apply epilogue, node gather)
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k3_contract|k3_gather_u|k4_apply_gather' -s 3 -c 5 -o gpurun_out/apply_v27 python microbench/time_kernels.py --config 5 --apply --reps 1 > gpurun_out/ncu73.log 2>&1; echo ncu $?

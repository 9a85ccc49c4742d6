# matrix-free apply (N1) at cfg5: total, per-kernel times, and a full capture of the apply-epilogue K3
timeout 200 python microbench/time_kernels.py --config 5 --apply --reps 3 | cut -c1-200
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/apply_launches.csv python microbench/time_kernels.py --config 5 --apply --reps 1 > /dev/null 2>&1; echo "launch rc=$?"
grep -E "gather_u|k3_contract<3, 2>|apply_gather" gpurun_out/apply_launches.csv | awk -F'","' '{print $5, $(NF)}' | tail -9
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k3_contract<3, 2>|k4_apply_gather|k3_gather_u' -s 3 -c 3 -o gpurun_out/apply_full python microbench/time_kernels.py --config 5 --apply --reps 1 > gpurun_out/ncu64.log 2>&1; echo ncu $?

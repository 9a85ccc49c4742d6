# K3 hand-over variants: old loop, old loop + fence-free ticket release, pipelined without frag_touch, pipelined with the wait after the tail DMMAs
for lib in microbench/libiga_IGA_EXPERIMENT_K3_NOPIPE.so microbench/libiga_IGA_EXPERIMENT_K3_NOPIPE_IGA_EXPERIMENT_K3_CHEAPREL.so microbench/libiga_IGA_EXPERIMENT_K3_NOTOUCH.so microbench/libiga_IGA_EXPERIMENT_K3_LATEWAIT.so; do
  echo $lib; IGA_LIB=$lib timeout 120 python microbench/time_kernels.py --config 5 --q 2 --reps 5 | grep -o "\"K3\": [0-9.]*"
done

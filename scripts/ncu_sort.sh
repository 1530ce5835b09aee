mkdir -p gpurun_out
CMD="python bench.py --config c4 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --eager"
$CMD > gpurun_out/plain_c4s.log 2>&1 && \
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
   -k 'regex:tile_sort_kernel|bin_entries' -s 6 -c 3 -o gpurun_out/ncu_sort_c4 $CMD > gpurun_out/ncu_sort.log 2>&1
echo "ncu rc=$?"

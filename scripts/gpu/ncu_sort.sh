# ncu --set full (with source) of the config-4 binning kernels: tile_sort and bin_entries (one launch each)
mkdir -p gpurun_out
CMD="python bench.py --config c4 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-secondary --eager"
$CMD > gpurun_out/ncu_sort_plain.log 2>&1 || { echo plain failed; exit 1; }
timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
   -k 'regex:tile_sort_kernel|bin_entries_kernel' -s 4 -c 2 -o gpurun_out/ncu_c4_sort $CMD > gpurun_out/ncu_sort.log 2>&1
echo "ncu rc=$?"; tail -2 gpurun_out/ncu_sort.log

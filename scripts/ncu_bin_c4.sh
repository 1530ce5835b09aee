mkdir -p gpurun_out
CMD="python bench.py --config c4 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --eager"
$CMD > gpurun_out/plain_c4b.log 2>&1 || { echo plain failed; exit 1; }
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
   -k 'regex:tile_sort|bin_entries|preprocess_fwd' -s 6 -c 3 -o gpurun_out/ncu_bin_c4 $CMD > gpurun_out/ncu_bin_c4.log 2>&1
echo "rc=$?"

mkdir -p gpurun_out
CMD="python bench.py --config c3 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --eager"
$CMD > gpurun_out/plain_c3.log 2>&1 && \
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
   -k 'regex:preprocess|emit_kernel|sort_pass|depth_fixup|tile_ranges' -s 200 -c 10 -o gpurun_out/ncu_c3_pre $CMD > gpurun_out/ncu_c3_pre.log 2>&1
echo "ncu rc=$?"

mkdir -p gpurun_out
CMD="python bench.py --config c3 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --eager"
$CMD > gpurun_out/plain_c3.log 2>&1 && \
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
   -k 'regex:raster_(fwd|bwd)_kernel<\(bool\)0' -s 64 -c 2 -o gpurun_out/ncu_c3 $CMD > gpurun_out/ncu_c3.log 2>&1
echo "ncu rc=$?"

mkdir -p gpurun_out
CMD="python bench.py --config c4 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --eager"
BSR_RASTER_G=1 $CMD > gpurun_out/plain_c4.log 2>&1 && \
BSR_RASTER_G=1 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
   -k 'regex:raster_(fwd|bwd)_kernel<\(bool\)0' -s 2 -c 2 -o gpurun_out/ncu_c4_G1 $CMD > gpurun_out/ncu_c4.log 2>&1
echo "ncu rc=$?"

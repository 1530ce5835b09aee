mkdir -p gpurun_out
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --eager"
for G in 1 4; do
  BSR_RASTER_G=$G $CMD > gpurun_out/plain_G$G.log 2>&1 && \
  BSR_RASTER_G=$G ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
     -k 'regex:raster_(fwd|bwd)_kernel<\(bool\)0' -s 4 -c 2 -o gpurun_out/ncu_G$G $CMD > gpurun_out/ncu_G$G.log 2>&1
  echo "G=$G ncu rc=$?"
done

# ncu --set full of the c4 raster kernels (one launch each), source-annotated
mkdir -p gpurun_out
CMD="python bench.py --config c4 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-secondary --eager"
$CMD > gpurun_out/ncu_c4_plain.log 2>&1 || { echo plain failed; tail gpurun_out/ncu_c4_plain.log; exit 1; }
timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
   -k 'regex:raster_(fwd|bwd)_kernel<\(bool\)0' -s 6 -c 2 -o gpurun_out/ncu_c4_raster $CMD > gpurun_out/ncu_c4.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/ncu_c4.log; ls -la gpurun_out/*.ncu-rep

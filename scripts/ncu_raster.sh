# ncu --set full of the raster kernels at c1 and c4 (after plain runs exit 0)
mkdir -p gpurun_out
for C in c1 c4; do
  S=5; [ $C = c4 ] && S=1
  CMD="python bench.py --config $C --steps $S --warmup 3 --no-cpu-baseline --no-e2e"
  $CMD > gpurun_out/plain_$C.log 2>&1 || { echo "plain $C failed"; tail -5 gpurun_out/plain_$C.log; continue; }
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
     -k 'regex:raster_(fwd|bwd)_kernel' -s 4 -c 2 -o gpurun_out/ncu_raster_$C $CMD > gpurun_out/ncu_raster_$C.log 2>&1
  echo "$C rc=$?"
done

# round-1 (session 4) evidence: c1 launch list + ncu full of the c1 step kernels, c3 colour chain
mkdir -p gpurun_out
C1="python bench.py --config c1 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e"
$C1 > gpurun_out/plain_c1.log 2>&1 || { echo "plain c1 failed"; tail -20 gpurun_out/plain_c1.log; exit 1; }
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c1.csv $C1 > gpurun_out/ncu_l_c1.log 2>&1
echo "launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
   -k 'regex:raster_(fwd|bwd)_kernel<\(bool\)0|ssim|preprocess_(fwd|bwd)|adam|bin_entries|tile_sort|replay' -s 40 -c 12 \
   -o gpurun_out/ncu_c1_full $C1 > gpurun_out/ncu_c1_full.log 2>&1
echo "full c1 rc=$?"
C3="python bench.py --config c3 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --eager"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
   -k 'regex:color_views|adam' -c 2 -o gpurun_out/ncu_c3_color $C3 > gpurun_out/ncu_c3_color.log 2>&1
echo "full c3 rc=$?"

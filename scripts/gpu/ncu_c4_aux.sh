# ncu --set full of the config-4 non-raster kernels (one launch each)
mkdir -p gpurun_out
CMD="python bench.py --config c4 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-secondary --eager"
$CMD > gpurun_out/ncu_aux_plain.log 2>&1 || { echo plain failed; exit 1; }
timeout 1500 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
   -k 'regex:tile_sort|bin_entries|preprocess_bwd_kernel|prebwd_geom|preprocess_fwd|ssim|replay_bwd' -s 10 -c 8 -o gpurun_out/ncu_c4_aux $CMD > gpurun_out/ncu_aux.log 2>&1
echo "ncu rc=$?"; tail -2 gpurun_out/ncu_aux.log

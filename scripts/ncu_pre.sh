mkdir -p gpurun_out
CMD="python bench.py --config c3 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --eager"
$CMD > gpurun_out/plain_c3p.log 2>&1 && \
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
   -k 'regex:preprocess_(fwd|bwd)_kernel|ssim' -s 40 -c 4 -o gpurun_out/ncu_pre_c3 $CMD > gpurun_out/ncu_pre.log 2>&1
echo "ncu rc=$?"

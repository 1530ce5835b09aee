mkdir -p gpurun_out
CMD="python bench.py --config c1 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain_c1l.log 2>&1 || { echo plain failed; exit 1; }
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
   -k 'regex:ssim' -s 6 -c 2 -o gpurun_out/ncu_loss $CMD > gpurun_out/ncu_loss.log 2>&1
echo "rc=$?"

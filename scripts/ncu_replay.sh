mkdir -p gpurun_out
C1="python bench.py --config c1 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
$C1 > gpurun_out/plain_c1.log 2>&1 || { echo "plain failed"; exit 1; }
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
   -k 'regex:replay_(fwd|bwd)' -s 6 -c 2 -o gpurun_out/ncu_replay $C1 > gpurun_out/ncu_replay.log 2>&1
echo "rc=$?"

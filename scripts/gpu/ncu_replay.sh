# ncu --set full of the config-4 fp64 replay kernels (forward and backward, one launch each)
mkdir -p gpurun_out
CMD="python bench.py --config c4 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-secondary --eager"
$CMD > gpurun_out/ncu_rp_plain.log 2>&1 || { echo plain failed; exit 1; }
timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
   -k 'regex:replay_' -s 6 -c 2 -o gpurun_out/ncu_c4_replay $CMD > gpurun_out/ncu_rp.log 2>&1
echo "ncu rc=$?"; tail -2 gpurun_out/ncu_rp.log
